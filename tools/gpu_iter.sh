#!/bin/bash
# Development loop on the GPU box: K2 parity subset, then timing (and phase profile) on config 4.
#   tools/gpu_iter.sh [pytest -k expr] [config]
K=${1:-"wavefront or families or edge or repeatable"}
CFG=${2:-geoknn_1m}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/iter_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/iter_tests.log
timeout 300 python tools/quick_perf.py $CFG - wavefront 50 > gpurun_out/iter_perf.log 2>&1
echo "perf exit $?" >> gpurun_out/iter_perf.log
POBK_K2_PROFILE=1 timeout 300 python tools/quick_perf.py $CFG - wavefront 50 > gpurun_out/iter_prof.log 2>&1
tail -3 gpurun_out/iter_tests.log; cat gpurun_out/iter_perf.log; grep "k2 prof" gpurun_out/iter_prof.log | tail -2
