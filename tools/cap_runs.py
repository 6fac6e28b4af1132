"""SURVEY.md §8(d) time-to-tolerance protocol for configs 3-5 beyond tol 0.1 (GPU only): the sweeps
and time to RSE < 1e-2, and a run to the 5e5-sweep cap at tol 1e-6 (time-to-1e-6
= "Inf" when the cap is reached), with the RSE at the cap and nnz-updates/s.  Writes markdown.

    python tools/cap_runs.py [out.md] [cap]
"""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2401_00672_b200 as pk
from workloads import gen

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/cap_runs.md"
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 500000
rows = []
for name in ["lap3d7_64", "geoknn_1m", "batch9pt_1024"]:
    systems = [gen.make(name, b) for b in range(8)] if name == "batch9pt_1024" else [gen.make(name)]
    tr = pk.half_gpu_tile_rows(systems[0].m) if len(systems) > 1 else 0
    plans = [pk.Plan.from_system(s, tile_rows=tr) for s in systems]
    fs = [torch.from_numpy(s.f).cuda() for s in systems]
    xst = [torch.from_numpy(s.x_star).cuda() for s in systems]
    xs = [torch.zeros(s.m, dtype=torch.float64, device="cuda") for s in systems]
    for tol, ms in ((1e-2, cap), (1e-6, cap)):
        for x in xs:
            x.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = pk.solve_batch(plans, fs, xs, xst, tol=tol, max_sweeps=ms, stop="rse")
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        sw = [r.sweeps for r in reps]
        conv = all(r.termination == 0 for r in reps)
        upd = sum(r.sweeps * p.nnz for r, p in zip(reps, plans))
        rows.append((name, len(systems), tol, ms, f"{min(sw)}-{max(sw)}" if len(set(sw)) > 1 else str(sw[0]),
                     "yes" if conv else "no (cap)", max(r.final_value for r in reps), t, upd / t / 1e9,
                     f"{t:.3f} s" if conv else "Inf"))
        print(rows[-1], flush=True)
    for p in plans:
        p.close()
lines = ["# Time-to-tolerance beyond 0.1 (configs 3-5, 1x B200, GPU only; SURVEY.md §8(d))", "",
         "`pobk_solve_batch` from x0 = 0, RSE checked every sweep; config 5: 8 systems per GPU on two lanes.  "
         "Time-to-tolerance is \"Inf\" when the cap is reached (the paper's convention, PAPER.md:366).", "",
         "| config | systems | tol | cap | sweeps | converged | RSE at stop (max) | wall (s) | G nnz-upd/s | time-to-tol |",
         "|---|---:|---:|---:|---:|---|---:|---:|---:|---|"]
for r in rows:
    lines.append(f"| {r[0]} | {r[1]} | {r[2]:g} | {r[3]} | {r[4]} | {r[5]} | {r[6]:.3e} | {r[7]:.2f} | {r[8]:.1f} | {r[9]} |")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
