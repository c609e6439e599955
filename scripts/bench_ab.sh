#!/bin/bash
# A/B of bounded config-3 bench runs (512^3, 8 slabs): per-sweep timed rate, kernel roofline, halo.
# VARIANTS="label:ENV=..,ENV=.." ; SWEEPS (cap), STEPS, WARMUP
cd "${GRAFT_REPO_ROOT:-.}"
for rep in $(seq ${REPS:-2}); do
for v in ${VARIANTS:-graph:BS_PERSIST=0 stream:BS_PERSIST=1}; do
  label=${v%%:*}; envs=${v#*:}
  env ${envs//,/ } timeout 600 python bench.py --max-outer ${SWEEPS:-40} --steps ${STEPS:-30} --warmup ${WARMUP:-5} \
     --no-cpu --no-config2 ${EXTRA} 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.readline()
try:
  d=json.loads(l)
except Exception:
  print('$label FAILED', l[:300]); sys.exit()
r=d['roofline']; h=d['halo']
print('$label', 'value %.2f Gpts/s' % d['value'], 'ms/step %.2f' % d['ms_per_step'], 'kernel %.1f us frac %.3f share %.3f' % (r['avg_launch_us'], r['frac'], r['share_of_step']),
      'halo %.1f us' % (h['avg_us'] or 0), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'], 'launches', d['gpu_launches'])
"
done
done
