#!/bin/bash
# pobk_solve_batch_host: the batch tests and the config-5 bench line (e2e through the host batch call)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "batch" > gpurun_out/r02i_batch_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02i_batch_tests.log
timeout 900 python bench.py --config batch9pt_1024 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02i_bench_c5_host.json 2> gpurun_out/r02i_bench_c5_host.err
tail -3 gpurun_out/r02i_batch_tests.log; cat gpurun_out/r02i_bench_c5_host.json; tail -5 gpurun_out/r02i_bench_c5_host.err
