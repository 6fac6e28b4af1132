#!/bin/bash
# Round-2 final evidence (session h): GPU suite, smoke, bench lines (config 4, config 5), the
# configs table, the ncu launch list of the bench and one ncu --set full capture of the K2 sweep.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02h_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02h_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02h_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err
timeout 900 python bench.py --config batch9pt_1024 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02h_bench_c5.json 2> gpurun_out/r02h_bench_c5.err
timeout 1500 python tools/configs_table.py gpurun_out/r02h_configs.md > gpurun_out/r02h_configs.log 2>&1
timeout 900 python tools/multi_rhs_perf.py geoknn_1m 50 > gpurun_out/r02h_multi_rhs_c4.log 2>&1
timeout 900 python tools/thr_perf.py > gpurun_out/r02h_thr_perf.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02h_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02h_ncu_launch.log 2>&1
timeout 1200 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k2_sweeps -s 3 -c 1 -o gpurun_out/r02h_k2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02h_ncu_full.log 2>&1
tail -3 gpurun_out/r02h_pytest_gpu.log; tail -1 gpurun_out/r02h_smoke.log; cat gpurun_out/r02h_bench.json; cat gpurun_out/r02h_bench_c5.json; cat gpurun_out/r02h_configs.md
