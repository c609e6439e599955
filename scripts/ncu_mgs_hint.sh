#!/bin/bash
# DRAM bytes per GMRES pointwise pass with and without the L2 policy (ncu with
# --cache-control none so the pass-to-pass L2 reuse stays visible).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for lib in libbsgpu_hint1.so libbsgpu.so; do
  BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 600 ncu --clock-control none --cache-control none \
    -k regex:k_point -c 500 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
    --log-file gpurun_out/ncu_mgs_$lib.csv python scripts/prof_gmres.py 256 30 > gpurun_out/ncu_mgs_$lib.log 2>&1
  echo "$lib rc=$?"
done
