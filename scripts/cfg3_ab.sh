#!/bin/bash
# A/B of library builds on a bounded config-3 run (512^3, 8 slabs, 30 sweeps): LIBS="a.so b.so" (in _lib/).
cd "${GRAFT_REPO_ROOT:-.}"
for lib in ${LIBS}; do
  BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 300 python bench.py --workload config3 --n 512 --steps 1 --warmup 0 \
    --max-outer ${SWEEPS:-30} 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$lib', round(d['time_to_solution_s'],3), 's', d['outer_sweeps'], d['inner_iterations_total'], round(d['stencil_gpts_per_s'],2), 'Gpts/s')"
done
