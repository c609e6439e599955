#!/bin/bash
# z-chunked tiling at 256^3 (BS_ZCHUNK): standalone residual / Jacobi / SpMV sweeps and the config-2 CG solve
cd "${GRAFT_REPO_ROOT:-.}"
for zc in ${ZCS:-0 128 64 0}; do
  echo "== BS_ZCHUNK=$zc"
  BS_ZCHUNK=$zc timeout 300 python scripts/time_sweeps.py 256
  BS_ZCHUNK=$zc timeout 300 python bench.py --workload config2 --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('config2', round(d['value'],2), 'Gpts/s', round(d['kernel_us']/1e3,2), 'ms kernel', 'frac', round(d['roofline_frac'],3))"
done
