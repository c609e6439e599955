#!/bin/bash
# Final tree: smoke + every GPU test; then the async stall diagnostic with SM clocks sampled every 100 ms
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final2_smoke.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/final2_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final2_pytest_gpu.log
tail -3 gpurun_out/final2_smoke.log gpurun_out/final2_pytest_gpu.log
nvidia-smi --query-gpu=timestamp,clocks.sm,pstate,utilization.gpu,power.draw --format=csv,noheader -lms 100 > gpurun_out/stall_clocks.csv 2>&1 &
SMI=$!
for i in 1 2 3 4 5; do
  date +"%Y/%m/%d %H:%M:%S.%3N start $i" >> gpurun_out/diag_async_v3.log
  timeout 120 python scripts/diag_async_stall.py 32 >> gpurun_out/diag_async_v3.log 2>&1
done
kill $SMI
cat gpurun_out/diag_async_v3.log
