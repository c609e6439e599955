#!/bin/bash
# A/B: persistent CG kernel vs the CUDA-graph path on the config-2 bench.
cd "${GRAFT_REPO_ROOT:-.}"
for mode in ${MODES:-0 1 0 1}; do
  BS_PERSIST=$mode timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('persist=$mode', round(d['value'],2), 'Gpts/s', round(d['ms_per_step'],2), 'ms', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
