#!/bin/bash
# Round evidence on the GPU box: full GPU suite, bench line, per-config table, ncu launch list,
# ncu --set full of K2 (config 4).
TAG=${1:-r01e}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench exit $?"
cat gpurun_out/${TAG}_bench.json
timeout 1500 python tools/configs_table.py gpurun_out/${TAG}_configs.md > gpurun_out/${TAG}_configs.log 2>&1; echo "configs exit $?"
timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_b_small.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches exit $?"
timeout 600 python tools/prof_k2.py geoknn_1m wavefront 10 > gpurun_out/${TAG}_prof_plain.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k2_sweeps -s 1 -c 1 -o gpurun_out/${TAG}_k2 \
    python tools/prof_k2.py geoknn_1m wavefront 10 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full exit $?"
