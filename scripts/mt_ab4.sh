#!/bin/bash
# A/B of the sweep launch shape on bounded config-4 (async) runs: rate per inner iteration.
cd "${GRAFT_REPO_ROOT:-.}"
run() {
  env "$@" timeout 300 python bench.py --workload config4 --n 512 --steps 1 --warmup 0 --max-outer ${SWEEPS:-400} 2>&1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$*', round(d['time_to_solution_s'],3), 's', d['outer_sweeps'], d['inner_iterations_total'], round(d['stencil_gpts_per_s'],2), 'Gpts/s')"
}
for rep in 1 2; do
  run BS_SWEEP_TILES=1
  run BS_SWEEP_PER_SM=3
done
