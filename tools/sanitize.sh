#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over tools/sanitize_cases.py: every
# kernel family at small shapes.  Logs to gpurun_out/sanitize_<tool>.log; run on the GPU box:
#   gpurun -- bash tools/sanitize.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -c 'ERROR SUMMARY\|=========' gpurun_out/sanitize_$tool.log) $(grep 'ERROR SUMMARY' gpurun_out/sanitize_$tool.log | tail -1)"
done
