"""Development: where config 4's end-to-end time goes (pobk_solve_host vs the device solve vs the
bare pinned copies).  python tools/e2e_breakdown.py [workload] [steps]"""
import sys
import time

import numpy as np
import torch

import paper_2401_00672_b200 as pk
from workloads import gen

name = sys.argv[1] if len(sys.argv) > 1 else "geoknn_1m"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
s = gen.make(name, 0)
plan = pk.Plan.from_system(s)
dev = torch.device("cuda", 0)
f, xs = torch.from_numpy(s.f).to(dev), torch.from_numpy(s.x_star).to(dev)
x = torch.zeros(s.m, dtype=torch.float64, device=dev)
hf = torch.from_numpy(s.f).pin_memory()
hxs = torch.from_numpy(s.x_star).pin_memory()
hx = [torch.zeros(s.m, dtype=torch.float64).pin_memory() for _ in range(3 * steps + 12)]
use = iter(range(len(hx)))
d3 = torch.empty(3 * s.m, dtype=torch.float64, device=dev)


def timed(fn, n=steps):
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n):
        fn(i)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


def dev_solve(i):
    x.zero_()
    plan.solve(f, x, xs, tol=0.1, stop="rse")


def host_solve(i):
    plan.solve_host(hf.numpy(), hx[next(use)].numpy(), hxs.numpy(), tol=0.1, stop="rse")


def copies(i):
    d3[: s.m].copy_(hf, non_blocking=True)
    d3[s.m: 2 * s.m].copy_(hx[i], non_blocking=True)
    d3[2 * s.m:].copy_(hxs, non_blocking=True)
    hx[i].copy_(d3[: s.m], non_blocking=True)
    torch.cuda.current_stream().synchronize()


def h2d_only(i):
    d3[: s.m].copy_(hf, non_blocking=True)
    d3[s.m: 2 * s.m].copy_(hx[i], non_blocking=True)
    d3[2 * s.m:].copy_(hxs, non_blocking=True)
    torch.cuda.current_stream().synchronize()


for lab, fn in (("device solve", dev_solve), ("host solve (pobk_solve_host)", host_solve), ("copies 24 MB in + 8 MB out", copies),
                ("copies 24 MB in", h2d_only)):
    ms = timed(fn)
    print(f"{lab:32s} {ms:8.3f} ms")
print("h2d GB/s", 3 * 8 * s.m / timed(h2d_only) / 1e6)
