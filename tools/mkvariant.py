"""Development: build a K2 source variant into tools/variants/libpobk_<name>.so.
python tools/mkvariant.py NAME EDITS.py  -- EDITS.py defines EDITS = [(old, new), ...] applied to
k2_wavefront.cu in a scratch copy of the package (the repo's sources are untouched)."""
import os, runpy, shutil, subprocess, sys

name, edits = sys.argv[1], runpy.run_path(sys.argv[2])["EDITS"]
here = os.path.dirname(os.path.abspath(__file__))
root = os.path.dirname(here)
dst = f"/tmp/var_{name}"
shutil.rmtree(dst, ignore_errors=True)
shutil.copytree(os.path.join(root, "paper_2401_00672_b200"), os.path.join(dst, "paper_2401_00672_b200"),
                ignore=shutil.ignore_patterns("_build", "*.so", "__pycache__"))
shutil.copytree(os.path.join(root, "include"), os.path.join(dst, "include"))
p = os.path.join(dst, "paper_2401_00672_b200", "csrc", "cuda", "k2_wavefront.cu")
s = open(p).read()
for old, new in edits:
    assert s.count(old) == 1, f"edit anchor not unique/found: {old[:80]!r}"
    s = s.replace(old, new)
open(p, "w").write(s)
env = dict(os.environ, POBK_BUILD_OUT=os.path.join(here, "variants", f"libpobk_{name}.so"),
           POBK_BUILD_DIR=os.path.join(dst, "_build"), POBK_PTXAS_V="1")
out = subprocess.run([sys.executable, os.path.join(dst, "paper_2401_00672_b200", "build.py")], env=env,
                     capture_output=True, text=True)
lines = [l for l in (out.stdout + out.stderr).splitlines() if "error" in l or "k2_sweeps" in l or "spill" in l
         or "registers" in l or "linked" in l]
print("\n".join(lines[-12:]))
sys.exit(out.returncode)
