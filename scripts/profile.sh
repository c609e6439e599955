#!/bin/bash
# ncu evidence for profiles/: launch list of a short bench run + one full capture of the sweep kernels.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/plain_bench.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launches.log 2>&1
python scripts/prof_cg.py 256 20 > gpurun_out/plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 12 -c 3 -o gpurun_out/prof_full \
      python scripts/prof_cg.py 256 20 > gpurun_out/ncu_full.log 2>&1
echo "profile done"
