#!/bin/bash
# Final build of the round (K1E incl. the residual-ordered loop): GPU suite, smoke, bench config 4.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02t_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02t_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02t_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02t_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02t_bench.json 2> gpurun_out/r02t_bench.err
tail -3 gpurun_out/r02t_pytest_gpu.log; tail -1 gpurun_out/r02t_smoke.log; cat gpurun_out/r02t_bench.json
