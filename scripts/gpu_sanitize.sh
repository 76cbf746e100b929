#!/bin/bash
# compute-sanitizer over every kernel family (scripts/sanitize_run.py); logs to gpurun_out/san_*.log
mkdir -p gpurun_out
python scripts/sanitize_run.py all > gpurun_out/san_plain.log 2>&1; echo "plain rc $?"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_run.py all > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc $? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_$tool.log | tail -1)"
done
