#!/bin/bash
# A/B of environment settings on the config-2 bench: ENVS="BS_ZCHUNK=128 BS_ZCHUNK=256 ..." ("-" = none).
cd "${GRAFT_REPO_ROOT:-.}"
for e in ${ENVS}; do
  if [ "$e" = "-" ]; then envs=""; else envs="${e//,/ }"; fi
  env $envs timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$e', round(d['value'],2), 'Gpts/s', round(d['ms_per_step'],2), 'ms', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
