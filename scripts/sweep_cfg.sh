#!/bin/bash
# Explore NSTAGE variants x z-chunk depths on the config-2 bench (no CPU/e2e legs).
cd "${GRAFT_REPO_ROOT:-.}"
for lib in ${LIBS:-libbsgpu.so libbsgpu_ab10.so libbsgpu_ab6.so}; do
  for zc in ${ZCS:-0 64 256}; do
    BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib BS_ZCHUNK=$zc timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e 2>&1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$lib zc=$zc', round(d['value'],2), 'S1', round(d['roofline']['frac'],3), round(d['roofline']['avg_launch_us'],1), 'S2', round(d['roofline_s2']['frac'],3), round(d['roofline_s2']['avg_launch_us'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 
  done
done
