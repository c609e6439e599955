#!/bin/bash
# A/B of the CG run path on a bounded config-3 run (512^3, 8 slabs): BS_PERSIST=0 (graph), 1 (default), 2 (tile loops)
cd "${GRAFT_REPO_ROOT:-.}"
for mode in ${MODES:-0 2 0 2}; do
  BS_PERSIST=$mode timeout 300 python bench.py --workload config3 --n 512 --steps 1 --warmup 0 \
    --max-outer ${SWEEPS:-30} 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('persist=$mode', round(d['time_to_solution_s'],3), 's', d['outer_sweeps'], d['inner_iterations_total'], round(d['stencil_gpts_per_s'],2), 'Gpts/s')"
done
