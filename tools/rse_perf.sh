#!/bin/bash
# Development: config-4 us/sweep with the RSE stop checked every sweep (the bench's setting) for
# several libpobk.so variants.  tools/rse_perf.sh "base ru8 ..."
for V in $1; do
  L=paper_2401_00672_b200/libpobk.so; [ $V != base ] && L=tools/variants/libpobk_$V.so
  W="bash tools/with_lib.sh $L 600"; [ $V = base ] && W="timeout 600"
  echo "== $V"; $W python tools/quick_perf.py geoknn_1m - wavefront 50 2>&1 | grep '"stop"'
done
