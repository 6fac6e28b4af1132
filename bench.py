"""POBK bench: nnz-updates/s and time-to-tolerance of the orthogonal-category Kaczmarz sweep on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config geoknn_1m] [--impl reference]
    (N > 1: python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N)

One STEP = one full pobk_solve of one batch of synthetic input: permute-in (Eq 3.1), sweeps of the
category schedule (Alg 5 loop) until RSE < tol checked every
sweep, permute-out.  Preprocessing (RCM + partition) runs once per system before the
timed region, like the paper's separate Table 1 timing.  Workload (BASELINE.json configs[3],
`geoknn_1m`): the largest single-system config, 1M-point kNN FEM-like matrix, 16.6M nnz, fp64.
Tolerance 1e-1 (1e-6 is unreachable within the paper's 5e5-sweep cap on this
config at row granularity; the protocol fixes 1e-1 for configs 3-5).

  value      = sum over ranks of nnz x sweeps / max-over-ranks device time of the K steps
  e2e        = the same metric through pobk_solve_host (pinned host f, x0, x*; H2D + D2H inside);
               batched configs through pobk_solve_batch_host (copies overlapped with other systems' sweeps)
  roofline   = the sweep kernel: algorithmic bytes B = 12 nnz + 12 m per sweep
               x sweeps / its CUDA-event time, against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline = the oracle (plain C, 1 core) on a bounded sample of the same workload
Multi-GPU: every rank solves its own independent systems (config 4: the same matrix with the rank's
own x*; --config batch9pt_1024: the batched config 5, systems rank*8 .. rank*8+7, 8 per GPU): weak
scaling, no data-path collective; NCCL only for the barrier, the max-over-ranks time and the
all_gather of per-system reports (C1) printed under "systems".
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TOL = {"lap2d5_32": 1e-6, "randband_20k": 1e-6, "lap3d7_64": 1e-1, "geoknn_1m": 1e-1, "batch9pt_1024": 1e-1}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="geoknn_1m")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="budget of the oracle sample")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, gpu: int):
        self.gpu, self.samples, self.proc, self.thread = gpu, [], None, None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_sample(s, seconds: float):
    """The oracle (plain C sweep, oracle/c/pobk_oracle.c) as it stands, 1 core, on a bounded sample
    of the same workload: its own preprocessing (untimed), then whole sweeps from x0 = 0 until the
    time budget; returns nnz-updates/s over the timed sweeps."""
    import oracle as O
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except Exception:
        pass
    t0 = time.time()
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    t_pre = time.time() - t0
    f_t = O.permute_vector(s.f, pre.perm)
    x_t = np.zeros(s.m)
    n = 0
    t0 = time.perf_counter()
    while True:
        O.sweep(pre, f_t, x_t, 1)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds or n >= 100000:
            break
    return {"value": s.nnz * n / el, "unit": "nnz-updates/s", "cores": 1, "kind": "oracle",
            "sample": f"{n} full sweeps of {s.name} from x0=0 (oracle preprocessing {t_pre:.1f}s untimed), "
                      f"{el:.1f}s, oracle/c/pobk_oracle.c row-by-row Eq 1.2, 1 pinned core of '{cpu_model()}'",
            "seconds_per_sweep": el / n}


def run_reference(a):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from workloads import gen
    s = gen.make(a.config)
    import oracle as O
    pre = O.preprocess(s.m, s.indptr, s.indices, s.data)
    f_t = O.permute_vector(s.f, pre.perm)
    # each step: a bounded sample of the solve -- a fixed number of oracle sweeps from x0 = 0
    probe = time.perf_counter()
    O.sweep(pre, f_t, np.zeros(s.m), 1)
    t1 = time.perf_counter() - probe
    per_step = max(1, int(min(20.0, 120.0 / max(1, a.steps + a.warmup)) / t1))
    for _ in range(a.warmup):
        O.sweep(pre, f_t, np.zeros(s.m), per_step)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        O.sweep(pre, f_t, np.zeros(s.m), per_step)
    el = time.perf_counter() - t0
    val = s.nnz * per_step * a.steps / el
    line = {"metric": "POBK nnz-updates/s (time-to-tolerance sweep)", "value": val, "unit": "nnz-updates/s",
            "impl": "reference", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": el / a.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": s.name if a.config != "batch9pt_1024" else f"{a.config} x8 per GPU", "m": s.m,
                       "nnz": s.nnz, "tol_rse": TOL[a.config], "stop": "rse",
                       "sample": "the same nnz-update (one row projection per stored nonzero per sweep) on the "
                                 "oracle, per-step sweep count bounded to ~20 s"},
            "cpu_baseline": {"value": val, "unit": "nnz-updates/s", "cores": 1, "kind": "oracle",
                             "sample": f"{per_step} oracle sweeps per step of {s.name} from x0=0 (the oracle as it "
                                       f"stands: oracle/c/pobk_oracle.c, 1 core of '{cpu_model()}')"},
            "e2e": {"value": val, "unit": "nnz-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    import torch
    import torch.distributed as dist

    import paper_2401_00672_b200 as pk
    from workloads import gen

    rank, world, local = dist_env()
    assert world == a.gpus or (world == 1 and a.gpus == 1), "launch N>1 with torchrun --nproc-per-node N"
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    tol = TOL[a.config]

    # ---- inputs (synthetic, BASELINE.json configs) and preprocessing: once, untimed.  Every rank
    #      solves its own systems: config 5 ids rank*8 .. rank*8+7; single-system configs system
    #      `rank` (the same matrix, its own x*: gen.CONFIGS)
    ids = [rank]
    if a.config == "batch9pt_1024":
        ids = [rank * 8 + b for b in range(8)]   # 8 independent systems per GPU
    systems = [gen.make(a.config, i) for i in ids]
    # batched systems: half-GPU tilings, so pobk_solve_batch runs two systems side by side
    tile_rows = pk.half_gpu_tile_rows(systems[0].m, local) if a.config == "batch9pt_1024" and a.kernel == "auto" else 0
    plans = [pk.Plan.from_system(s, kernel=a.kernel, device=local, tile_rows=tile_rows) for s in systems]
    fs = [torch.from_numpy(s.f).to(dev) for s in systems]
    xss = [torch.from_numpy(s.x_star).to(dev) for s in systems]
    xs = [torch.zeros(s.m, dtype=torch.float64, device=dev) for s in systems]
    stream = torch.cuda.current_stream()

    def step():
        for x in xs:
            x.zero_()
        if len(plans) > 1:  # one pobk_solve_batch call (concurrent lanes when the tiling allows)
            return pk.solve_batch(plans, fs, xs, xss, tol=tol, max_sweeps=500000, stop="rse")
        return [plans[0].solve(fs[0], xs[0], xss[0], tol=tol, max_sweeps=500000, stop="rse")]

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    all_reps = []
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(a.steps):
            all_reps.extend(step())
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t = ev0.elapsed_time(ev1) * 1e-3
    updates = float(sum(r.sweeps * p.nnz for r, p in zip(all_reps, plans * a.steps)))
    sweep_t = sum(r.sweep_seconds for r in all_reps)
    sweeps = sum(r.sweeps for r in all_reps)
    launches = sum(r.launches for r in all_reps)

    # ---- e2e: the public C-ABI call with host buffers (pinned), copies inside the timed region
    hf = [torch.from_numpy(s.f).pin_memory().numpy() for s in systems]
    hxs = [torch.from_numpy(s.x_star).pin_memory().numpy() for s in systems]
    # x is in/out (x0 in): one pinned x0 = 0 buffer per step and system, zeroed before the timed
    # region, unless that exceeds 512 MB (then one set, re-zeroed on the host inside the loop)
    per_step = a.steps * sum(8 * s.m for s in systems) <= (512 << 20)
    nset = a.steps if per_step else 1
    hx = [[torch.zeros(s.m, dtype=torch.float64).pin_memory().numpy() for s in systems] for _ in range(nset)]
    e2e_reps = []
    # untimed warm-up of the host path (its first call allocates the plans' staging buffers)
    for _ in range(a.warmup):
        hw = [np.zeros(s.m) for s in systems]
        if len(plans) > 1:
            pk.solve_batch_host(plans, hf, hw, hxs, tol=tol, max_sweeps=500000, stop="rse")
        else:
            plans[0].solve_host(hf[0], hw[0], hxs[0], tol=tol, stop="rse")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if len(plans) > 1:
        # batched systems: one pobk_solve_batch_host call per step on the pinned host vectors (its
        # internal copy streams move the other systems' inputs in and the finished solutions out
        # while systems solve on the lanes); all inside the timed region
        for st in range(a.steps):
            hxs_t = hx[st if per_step else 0]
            if not per_step:
                for v in hxs_t:
                    v[:] = 0.0
            e2e_reps.extend(pk.solve_batch_host(plans, hf, hxs_t, hxs, tol=tol, max_sweeps=500000, stop="rse"))
    else:
        for st in range(a.steps):
            for p, f, x, xst in zip(plans, hf, hx[st if per_step else 0], hxs):
                if not per_step:
                    x[:] = 0.0
                e2e_reps.append(p.solve_host(f, x, xst, tol=tol, stop="rse"))
    torch.cuda.synchronize()
    t_e2e = time.perf_counter() - t0
    e2e_updates = float(sum(r.sweeps * p.nnz for r, p in zip(e2e_reps, plans * a.steps)))
    err = max(float(np.linalg.norm(x.cpu().numpy() - s.x_star) / np.linalg.norm(s.x_star)) for x, s in zip(xs, systems))

    from paper_2401_00672_b200 import driver
    # C1: per-system reports of the last timed step gathered from every rank (all_gather)
    agg = driver.gather_reports([driver.system_report(i, p.nnz, r) for i, p, r in zip(ids, plans, all_reps[-len(plans):])],
                                t, dev)
    if world > 1:
        t, t_e2e, sweep_t = (driver.max_over_ranks(v, dev) for v in (t, t_e2e, sweep_t))
        updates, e2e_updates = (driver.sum_over_ranks(v, dev) for v in (updates, e2e_updates))
    if rank != 0:
        dist.destroy_process_group()
        return 0

    s0 = systems[0]
    B = 12.0 * s0.nnz + 12.0 * s0.m          # algorithmic bytes per sweep
    peaks = measured_peaks()
    peak = peaks.get("hbm_gbs")
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy)" if peak else "fallback 6650 GB/s (B200_PROFILING.md)"
    peak = peak or 6650.0
    # sweep-kernel time: the sum of the per-solve sweep-kernel event spans -- unless the batch ran
    # on concurrent lanes (the spans overlap), then the timed region itself (all kernels of the
    # step; the sweep kernels are ~98% of it, profiles/*_launches.md)
    lanes = len(plans) > 1 and sweep_t > 1.05 * t
    kern_t = t if lanes else sweep_t
    # lanes pobk_solve_batch used (its rule: every plan K2, min(4, SMs / max tiles, systems))
    nlanes = None
    if len(plans) > 1:
        st_all = [p.layout_stats() for p in plans]
        if all(x["kernel"] == "wavefront" for x in st_all):
            sms = torch.cuda.get_device_properties(local).multi_processor_count
            nlanes = max(1, min(4, sms // max(x["ntiles"] for x in st_all), len(plans)))
        else:
            nlanes = 1
    l2_bytes = 126e6
    resident = B * len(systems) <= l2_bytes
    achieved = B * sweeps / kern_t / 1e9 if kern_t > 0 else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))  # {workload: {kernel, dram_bytes_per_sweep, source}}
            tj = tj.get(s0.name, {}) if "workload" not in tj else tj
            if tj.get("workload") == s0.name and tj.get("kernel") == all_reps[0].as_dict()["kernel"]:
                traffic = tj.get("dram_bytes_per_sweep")
        except Exception:
            pass
    stats = plans[0].layout_stats()
    line = {
        "metric": "POBK nnz-updates/s (time-to-tolerance sweep)",
        "value": updates / t,
        "unit": "nnz-updates/s",
        "n_gpus": world,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": t / a.steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": s0.name if a.config != "batch9pt_1024" else f"{a.config} x8 per GPU",
                   "m": s0.m, "nnz": s0.nnz, "systems_per_gpu": len(systems), "tol_rse": tol, "stop": "rse",
                   "sweeps_per_solve": all_reps[0].sweeps, "kernel": all_reps[0].as_dict()["kernel"],
                   "batch_lanes": nlanes,
                   "tiles": stats["ntiles"], "threads_per_cta": stats["threads"], "private_nnz_frac": round(stats["private_nnz_frac"], 4),
                   "nsteps": plans[0].nsteps, "bandwidth_rcm": plans[0].bw_after,
                   "preprocess_s": round(plans[0].preprocess_seconds, 3),
                   "l2": ("working set %.1f MB fits the 126 MB L2: L2-resident by design (no flush); the HBM "
                          "fraction below is not a bound for it" % (B * len(systems) / 1e6)) if resident else
                         ("inputs larger than L2 (A stream %.0f MB per GPU > 126 MB), no flush" % (B * len(systems) / 1e6)),
                   "time_to_tol_ms": sum(r.solve_seconds for r in all_reps) / len(all_reps) * 1e3,
                   "final_rse": all_reps[-1].final_value, "rel_err_vs_xstar": err},
        "e2e": {"value": e2e_updates / t_e2e, "unit": "nnz-updates/s",
                "h2d_bytes_per_step": int(sum(3 * 8 * s.m for s in systems)),
                "d2h_bytes_per_step": int(sum(8 * s.m for s in systems))},
        "gpu_launches": int(launches),
        "systems": [{"rank": pr["rank"], "ids": [r["id"] for r in pr["systems"]], "sweeps": [r["sweeps"] for r in pr["systems"]],
                     "final_rse": [r["final"] for r in pr["systems"]]} for pr in agg["ranks"]],
        "roofline": {"bound": "l2" if resident else "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "kernel": "sweep (" + all_reps[0].as_dict()["kernel"] + ")", "peak_source": peak_src,
                     "bytes_per_sweep": B, "us_per_sweep": kern_t / sweeps * 1e6,
                     "timing": "aggregate over the timed region (concurrent lanes)" if lanes else "sweep-kernel CUDA events"},
        "clocks": clk.summary(),
    }
    if world == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"] = oracle_sample(s0, a.cpu_seconds)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
