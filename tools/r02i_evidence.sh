#!/bin/bash
# Round-2 re-entry evidence (session i): GPU suite, smoke, bench lines (config 4, config 5), the
# ncu launch list of the bench and one ncu --set full capture of the K2 sweep.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02i_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02i_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02i_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02i_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err
timeout 900 python bench.py --config batch9pt_1024 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02i_bench_c5.json 2> gpurun_out/r02i_bench_c5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02i_bench_ref.json 2> gpurun_out/r02i_bench_ref.err
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02i_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02i_ncu_launch.log 2>&1
timeout 1200 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k2_sweeps -s 3 -c 1 -o gpurun_out/r02i_k2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02i_ncu_full.log 2>&1
tail -3 gpurun_out/r02i_pytest_gpu.log; tail -1 gpurun_out/r02i_smoke.log; cat gpurun_out/r02i_bench.json; cat gpurun_out/r02i_bench_c5.json; cat gpurun_out/r02i_bench_ref.json
