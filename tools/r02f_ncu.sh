#!/bin/bash
# r02f: the ncu launch list of the bench (config 4) and one ncu --set full capture of the K2 sweep
mkdir -p gpurun_out
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_ncu_launch.log 2>&1
timeout 1200 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k2_sweeps -s 3 -c 1 -o gpurun_out/r02f_k2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_ncu_full.log 2>&1
tail -2 gpurun_out/r02f_ncu_full.log
