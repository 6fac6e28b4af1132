#!/bin/bash
# Development: us/sweep of K2 on one config for several VSlice poll back-offs (POBK_K2_NAP, ns)
# and lane widths; optional ncu stall breakdown of one sweep kernel.
CFG=${1:-geoknn_1m}; NAPS=${2:-"0 64 200"}; VLS=${3:-"-1"}; NCU=${4:-0}
mkdir -p gpurun_out
for V in $VLS; do for N in $NAPS; do
  echo "== $CFG VL=$V NAP=$N"
  POBK_K2_VL=$V POBK_K2_NAP=$N timeout 300 python tools/quick_perf.py $CFG - wavefront 50 2>&1 | grep -E '"stop"|rror' | tail -2
done; done
if [ "$NCU" != "0" ]; then
  for V in $VLS; do
  POBK_K2_VL=$V timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none -k regex:k2_sweeps -c 1 -o gpurun_out/ncu_vl$V -f python tools/quick_perf.py $CFG - wavefront 20 > gpurun_out/ncu_vl$V.log 2>&1
  /usr/local/cuda/bin/ncu -i gpurun_out/ncu_vl$V.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for k,x in zip(h,v):
    if 'smsp__average_warp' in k and 'issue_stalled' in k and 'ratio' in k and x not in ('','0'):
        try:
            if float(x)>0.05: print(k,x)
        except: pass
    if k in ('gpu__time_duration.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','smsp__issue_active.avg.pct_of_peak_sustained_active'): print(k,x)
"
  done
fi
