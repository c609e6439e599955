#!/bin/bash
# Round evidence in one GPU call: smoke, GPU tests, bench, ncu launch list +
# full capture (profile.sh), GMRES block-scheduling A/B, bounded config-5 run
# at its full 1024^3 size.  Outputs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
bash scripts/gpu_check.sh
bash scripts/profile.sh
for sh in 0 1; do
  echo "BS_GMRES_SHARED=$sh" >> gpurun_out/ab_solo.log
  BS_GMRES_SHARED=$sh timeout 300 python scripts/prof_outer.py config5 512 4 2>&1 | tail -2 >> gpurun_out/ab_solo.log
done
timeout 900 python bench.py --workload config5 --n 1024 --steps 1 --warmup 0 --max-outer ${CFG5_SWEEPS:-100} \
  > gpurun_out/cfg5_1024.log 2>&1
echo "round_check done"
