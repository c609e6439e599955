#!/bin/bash
# A/B: multi-tile sweep CTAs with dynamic tile hand-out (default) vs one tile per CTA (BS_SWEEP_TILES=1).
cd "${GRAFT_REPO_ROOT:-.}"
for m in ${MODES:-1 0 1 0}; do
  BS_SWEEP_TILES=$m timeout 300 python bench.py --workload config3 --n 512 --steps 1 --warmup 0 --max-outer ${SWEEPS:-60} 2>&1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('tiles1=$m config3', round(d['time_to_solution_s'],3), 's', d['outer_sweeps'], d['inner_iterations_total'], round(d['stencil_gpts_per_s'],2), 'Gpts/s')"
done
