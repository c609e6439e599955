#!/bin/bash
# A/B of library builds on the config-2 bench: LIBS="a.so b.so ..." (in _lib/).
cd "${GRAFT_REPO_ROOT:-.}"
for lib in ${LIBS}; do
  BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$lib', round(d['value'],2), 'Gpts/s', round(d['ms_per_step'],2), 'ms', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
