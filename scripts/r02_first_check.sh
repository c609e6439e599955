#!/bin/bash
# Re-entry check: smoke + GPU tests, then a GMRES(30) cycle at 512^3 (one
# config-5 block at 1024^3 is 514^3) timed plain and as an ncu launch list.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/prof_gmres.py 512 30 > gpurun_out/gmres512.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/gmres512_launches.csv python scripts/prof_gmres.py 512 30 > gpurun_out/gmres512_ncu.log 2>&1
echo done
