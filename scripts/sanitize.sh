#!/bin/bash
# compute-sanitizer over scripts/sanitize_cases.py: memcheck, racecheck, synccheck (summaries to gpurun_out/)
cd "${GRAFT_REPO_ROOT:-.}"
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python scripts/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
done
