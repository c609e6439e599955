#!/bin/bash
# One segment of the config-5 solve at 1024^3 (scripts/run_cfg5.py): SEG=1 starts, SEG>1 resumes from the
# checkpoint the previous call left in /tmp/cfg5_ckpt on the same box.  Logs go to gpurun_out/cfg5_seg<SEG>.log.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
SEG=${SEG:-1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv,noheader > gpurun_out/cfg5_seg${SEG}_gpu.txt 2>&1
df -h /tmp | tail -1 >> gpurun_out/cfg5_seg${SEG}_gpu.txt
(while true; do nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader >> gpurun_out/cfg5_seg${SEG}_smi.csv; sleep 60; done) &
SMI=$!
if [ "$SEG" = "1" ]; then rm -rf /tmp/cfg5_ckpt; R=0; else R=1; fi
RESUME=$R SEG_BUDGET_S=${SEG_BUDGET_S:-3250} LOG_EVERY=${LOG_EVERY:-25} CKPT_DIR=/tmp/cfg5_ckpt \
  timeout 3450 python scripts/run_cfg5.py ${CFG5_N:-1024} > gpurun_out/cfg5_seg${SEG}.log 2> gpurun_out/cfg5_seg${SEG}.err
echo "rc=$?" >> gpurun_out/cfg5_seg${SEG}.log
kill $SMI
ls -la /tmp/cfg5_ckpt | head -40 >> gpurun_out/cfg5_seg${SEG}_gpu.txt
tail -4 gpurun_out/cfg5_seg${SEG}.log
