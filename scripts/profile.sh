#!/bin/bash
# ncu evidence for profiles/: launch list of a short bench run + one full
# capture of the dominant kernel (the persistent CG kernel over a whole
# 856-iteration config-2 solve).  Each ncu run only after the same command
# exited 0 without ncu.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/plain_bench.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launches.log 2>&1
python scripts/prof_persist.py 256 856 > gpurun_out/plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_cg_persistent -c 1 -o gpurun_out/prof_full \
      python scripts/prof_persist.py 256 856 > gpurun_out/ncu_full.log 2>&1
echo "profile done"
