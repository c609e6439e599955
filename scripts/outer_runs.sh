#!/bin/bash
# Supplemental outer-solve workloads (configs 3/4/5) on one GPU.  RUNS="config3:512 config5:256"
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for spec in ${RUNS:-config3:128 config4:128 config5:64}; do
  w=${spec%%:*}; n=${spec##*:}
  timeout ${RUN_TIMEOUT:-600} python bench.py --workload $w --n $n --steps 1 --warmup 0 >> gpurun_out/outer_runs.log 2>&1
  echo "$w n=$n rc=$?" >> gpurun_out/outer_runs.log
done
