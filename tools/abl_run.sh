#!/bin/bash
# Development: K2 us/sweep with ablation builds (wrong numerics; timing only), one config.
CFG=${1:-geoknn_1m}
echo "== base"; timeout 300 python tools/quick_perf.py $CFG - wavefront 50 2>&1 | grep '"stop": "none"'
for A in $2; do
  echo "== ABL=$A"
  timeout 300 bash tools/run_variant.sh tools/variants/libpobk_abl$A.so python tools/quick_perf.py $CFG - wavefront 50 2>&1 | grep '"stop": "none"'
done
