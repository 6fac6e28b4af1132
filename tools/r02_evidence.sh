#!/bin/bash
# Round-2 evidence on the GPU box: thr > 0 measurement, bench lines (config 4, config 5), the ncu
# launch list of the bench and one ncu --set full capture of the K2 sweep kernel.
mkdir -p gpurun_out
timeout 900 python tools/thr_perf.py > gpurun_out/r02_thr_perf.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
timeout 900 python bench.py --config batch9pt_1024 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu_launch.log 2>&1
timeout 1200 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k2_sweeps -s 3 -c 1 -o gpurun_out/r02_k2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu_full.log 2>&1
cat gpurun_out/r02_thr_perf.log; cat gpurun_out/r02_bench.json; cat gpurun_out/r02_bench_c5.json; tail -3 gpurun_out/r02_ncu_full.log
