#!/bin/bash
# K1E (sliced ELL for the launch path): the K1-touching GPU tests, then CSR vs ELL timings.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -k "fixed_sweeps_parity or kernel_families or stop_sweep_parity or thr_positive or edge_cases or nonfinite or relres_stop or residual_order or fully_orthogonal or sweep_offset" > gpurun_out/r02q_pytest_k1.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02q_pytest_k1.log
timeout 900 python tools/k1e_perf.py > gpurun_out/r02q_k1e_perf.log 2>&1; echo "exit $?" >> gpurun_out/r02q_k1e_perf.log
tail -3 gpurun_out/r02q_pytest_k1.log; cat gpurun_out/r02q_k1e_perf.log
