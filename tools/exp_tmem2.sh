#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -x tests/test_gpu_wavefront.py tests/test_gpu_parity.py -k "config4_full or config3_full or config5_full or kernel_families or long_rows or many_small or batch or stop_sweep_bench" > gpurun_out/tm2_pytest.log 2>&1; tail -3 gpurun_out/tm2_pytest.log
for V in r02f tm2; do echo "== $V"; bash tools/with_lib.sh tools/variants/libpobk_$V.so 300 python tools/knob_perf.py geoknn_1m 0 "DYN=0" 50 2>&1 | grep us_per | tail -1
  bash tools/with_lib.sh tools/variants/libpobk_$V.so 600 python bench.py --config batch9pt_1024 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', round(d['value']/1e9,1), 'G', d['roofline']['frac'])"; done
