#!/bin/bash
# Time K2 development variants (tools/variants/libpobk_exp<N>.so) on one config: us/sweep + RSE after 50 sweeps.
CFG=${CFG:-geoknn_1m}
mkdir -p gpurun_out
echo "== main"; timeout 300 python tools/quick_perf.py $CFG - wavefront 50 2>&1 | grep -E '"stop"' | tail -2
for E in "$@"; do
  echo "== EXP $E"
  bash tools/run_variant.sh tools/variants/libpobk_exp$E.so timeout 300 python tools/quick_perf.py $CFG - wavefront 50 2>&1 | grep -E '"stop"|rror' | tail -2
done
