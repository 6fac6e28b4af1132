#!/bin/bash
# K2 end-of-sweep RSE scan with the x~* values loaded into registers before the last task barrier
# (variants pfa: 16/8 double2 per thread at 256/512 threads, pfb: 12/6), built by tools/mkvariant.py
mkdir -p gpurun_out
for V in base pfa pfb; do
  W="bash tools/with_lib.sh tools/variants/libpobk_$V.so 300"; [ $V = base ] && W="timeout 300"
  echo "== $V"
  for C in geoknn_1m lap3d7_64; do $W env PYTHONPATH=. python tools/rse_us.py $C 0.1 2>&1 | tail -2; done
done > gpurun_out/r02i_rse_prefetch.log 2>&1
for V in base pfa pfb base; do
  W="bash tools/with_lib.sh tools/variants/libpobk_$V.so 300"; [ $V = base ] && W="timeout 300"
  echo "== $V"; $W env PYTHONPATH=. python tools/rse_us.py geoknn_1m 0.1 2>&1 | tail -2
done >> gpurun_out/r02i_rse_prefetch.log 2>&1
cat gpurun_out/r02i_rse_prefetch.log
