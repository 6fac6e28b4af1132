#!/bin/bash
# Development: K2 parity subset, then us/sweep for several boundary-slice lane widths (POBK_K2_VL).
#   tools/vl_sweep.sh "<pytest -k expr>" "<VL values>" "<configs>"
K=${1:-"wavefront or families"}
VLS=${2:-"0 4 8"}
CFGS=${3:-"geoknn_1m lap3d7_64 randband_20k"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
if [ "$K" != "-" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/iter_tests.log 2>&1
  echo "tests exit $?" >> gpurun_out/iter_tests.log
  tail -3 gpurun_out/iter_tests.log
fi
for C in $CFGS; do
  for V in $VLS; do
    echo "== $C VL=$V"
    POBK_K2_VL=$V timeout 300 python tools/quick_perf.py $C - wavefront 50 2>&1 | grep -E '"stop"|Error|error' | tail -2
  done
done
