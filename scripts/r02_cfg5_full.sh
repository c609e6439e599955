#!/bin/bash
# Config 5 (BASELINE configs[4]) at its full 1024^3 size on one B200, to
# convergence: progress every LOG_EVERY sweeps, final summary line.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/cfg5_gpu.txt 2>&1
(while true; do nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> gpurun_out/cfg5_smi.csv; sleep 60; done) &
SMI=$!
LOG_EVERY=${LOG_EVERY:-25} timeout ${CFG5_TIMEOUT:-19200} python scripts/run_cfg5.py 1024 > gpurun_out/cfg5_1024_full.log 2> gpurun_out/cfg5_1024_full.err
echo "rc=$?" >> gpurun_out/cfg5_1024_full.log
kill $SMI
