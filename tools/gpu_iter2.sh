#!/bin/bash
# Development loop on the GPU box: K2 parity subset, timing on configs 4/3/2, one traced sweep
# (phases + hops) on config 4.
K=${1:-"wavefront or families or edge or repeatable"}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/iter_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/iter_tests.log
tail -3 gpurun_out/iter_tests.log
for C in geoknn_1m lap3d7_64 randband_20k; do
  timeout 300 python tools/quick_perf.py $C - wavefront 50 2>&1 | grep -E '"stop"' | tail -2
done
timeout 300 python tools/k2_hops.py geoknn_1m 10 > gpurun_out/iter_hops.log 2>&1; cat gpurun_out/iter_hops.log | tail -8
timeout 120 python tools/k2_phases.py gpurun_out/k2_trace.bin 2>&1 | tail -12
