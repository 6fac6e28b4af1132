#!/bin/bash
# Development: K2 us/sweep of several libpobk.so variants (tools/variants/libpobk_<name>.so) on
# configs 4 and 3, plus the config-5 bench line's aggregate.  tools/variant_perf.sh "base s32 ..."
for V in $1; do
  echo "== $V"
  L=paper_2401_00672_b200/libpobk.so; [ $V != base ] && L=tools/variants/libpobk_$V.so
  W="bash tools/with_lib.sh $L 600"; [ $V = base ] && W="timeout 600"
  for C in geoknn_1m lap3d7_64; do $W python tools/knob_perf.py $C 0 "DYN=0" 2>&1 | tail -1; done
  $W python bench.py --config batch9pt_1024 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', round(d['value']/1e9,1), 'G', d['roofline']['frac'], d['config']['kernel'], d['config']['batch_lanes'])"
done
