#!/bin/bash
# thr > 0: ordered per-column scatter (default) vs the fp64-atomic scatter -- parity tests, timings
mkdir -p gpurun_out
timeout 900 python -m pytest -q tests/test_gpu_parity.py -k "thr_positive" > gpurun_out/thr_pytest.log 2>&1; tail -3 gpurun_out/thr_pytest.log
echo "== ordered"; timeout 900 python tools/thr_perf.py 2>&1 | grep '"thr": 0\.[0-9]*[1-9]'
echo "== atomic"; POBK_THR_ATOMIC=1 timeout 900 python tools/thr_perf.py 2>&1 | grep '"thr": 0\.[0-9]*[1-9]'
