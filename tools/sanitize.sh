#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_workload.py (GPU).
#   bash tools/sanitize.sh <outdir>
out=${1:-gpurun_out/sanitize}; mkdir -p $out
for tool in memcheck racecheck synccheck; do
  timeout 1800 compute-sanitizer --tool $tool --print-limit 50 --target-processes all \
    python tools/sanitize_workload.py > $out/$tool.txt 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|WORKLOAD' $out/$tool.txt | tr '\n' ' ')"
done
