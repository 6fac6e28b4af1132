#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py;
# summaries into gpurun_out/sanitize_<tool>.log
CS=/usr/local/cuda/bin/compute-sanitizer
for T in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $T --target-processes all --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_$T.log 2>&1
  echo "$T exit $?" >> gpurun_out/sanitize_$T.log
  echo "== $T"; grep -E "ERROR SUMMARY|SANITIZE-RUN|exit|Error|Hazard" gpurun_out/sanitize_$T.log | head -8
done
