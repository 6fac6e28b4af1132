#!/bin/bash
# Round-2 final evidence (last re-entry session: rebuilt in a fresh container from HEAD):
# GPU suite, smoke, bench lines (config 4, config 5), ncu launch list of the bench.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02n_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02n_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02n_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02n_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err
timeout 900 python bench.py --config batch9pt_1024 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02n_bench_c5.json 2> gpurun_out/r02n_bench_c5.err
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02n_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02n_ncu_launch.log 2>&1
tail -3 gpurun_out/r02n_pytest_gpu.log; tail -1 gpurun_out/r02n_smoke.log; cat gpurun_out/r02n_bench.json; cat gpurun_out/r02n_bench_c5.json
