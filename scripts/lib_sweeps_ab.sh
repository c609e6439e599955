#!/bin/bash
# A/B of library builds (LIBS, in _lib/): standalone sweeps at 256^3 and a bounded config-3 bench
cd "${GRAFT_REPO_ROOT:-.}"
for rep in 1 2; do for lib in ${LIBS}; do
  echo "== $lib"
  BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 300 python scripts/time_sweeps.py 256
  [ -z "$SLAB" ] || BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 300 python scripts/time_sweeps.py 512 512 64 | sed 's/^/slab 512x512x64 /'
  [ -n "$NOBENCH" ] || BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 600 python bench.py --max-outer 30 --steps 20 --warmup 5 --no-cpu --no-config2 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('config3 bounded', round(d['value'],2), 'Gpts/s', round(d['ms_per_step'],2), 'ms/step')"
done; done
