#!/bin/bash
# Round-2 (session f) evidence: GPU suite, smoke, bench lines (config 4, config 5), config-1 K3E
# timing against the previous build, the ncu launch list of the bench.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02f_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02f_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02f_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err
timeout 900 python bench.py --config batch9pt_1024 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_bench_c5.json 2> gpurun_out/r02f_bench_c5.err
for V in base r02f; do echo "== $V"; bash tools/with_lib.sh tools/variants/libpobk_$V.so 300 python tools/quick_perf.py lap2d5_32 - smem 20000 2>&1 | grep us_per | tail -2; done > gpurun_out/r02f_k3e.log
tail -3 gpurun_out/r02f_pytest_gpu.log; tail -1 gpurun_out/r02f_smoke.log; cat gpurun_out/r02f_bench.json; cat gpurun_out/r02f_bench_c5.json; cat gpurun_out/r02f_k3e.log
