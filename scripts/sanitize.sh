#!/bin/bash
# GPU box: run scripts/sanitize_cases.py under compute-sanitizer's memcheck,
# racecheck (shared-memory hazards) and synccheck; logs in gpurun_out/.
set -u
mkdir -p gpurun_out
N=${N:-40000}
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
    python scripts/sanitize_cases.py $N > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.log
done
