#!/bin/bash
# A/B of the CG run path on a bounded config-3 run (512^3, 8 slabs, SWEEPS sweeps):
# graph path (BS_PERSIST=0) vs the streaming persistent kernel (default), and library variants (LIBS)
cd "${GRAFT_REPO_ROOT:-.}"
run() {  # label, env...
  env "${@:2}" timeout 300 python bench.py --workload config3 --n 512 --steps 1 --warmup 0 --max-outer ${SWEEPS:-30} 2>&1 \
   | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$1', round(d['time_to_solution_s'],3), 's', d['outer_sweeps'], d['inner_iterations_total'], round(d['stencil_gpts_per_s'],2), 'Gpts/s')"
}
for rep in 1 2; do
  run graph BS_PERSIST=0
  run stream3 BS_PERSIST=1
  for lib in ${LIBS}; do run "stream:$lib" BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib BS_PERSIST=1; done
done
