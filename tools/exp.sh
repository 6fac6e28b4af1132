python tools/k2_trace.py geoknn_1m 10 20 2>&1 | grep -E "post:|us/sweep|boundary slice" > gpurun_out/exp0.log
for E in 1 4 5; do bash tools/run_variant.sh tools/variants/libpobk_exp$E.so python tools/k2_trace.py geoknn_1m 10 20 2>&1 | grep -E "post:|us/sweep|boundary slice" > gpurun_out/exp$E.log; done
for E in 0 1 4 5; do echo "== EXP $E"; cat gpurun_out/exp$E.log; done
