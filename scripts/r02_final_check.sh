#!/bin/bash
# Round-2 final evidence: PART=A smoke, every GPU test, the driver's bench command and the reference arm;
# PART=B the ncu launch list of a bounded bench run and --set full captures of the sweeps (scripts/round_bench.sh).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-r02v2}
if [ "${PART:-A}" = "A" ]; then
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/final_gpu.txt 2>&1
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final_smoke.log
  timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 --durations=10 > gpurun_out/final_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest_gpu.log
  tail -n 3 gpurun_out/final_smoke.log gpurun_out/final_pytest_gpu.log
  TAG=$TAG NO_NCU=1 bash scripts/round_bench.sh
  tail -c 600 gpurun_out/${TAG}_bench.log; tail -c 300 gpurun_out/${TAG}_ref.log
else
  TAG=$TAG NO_BENCH=1 bash scripts/round_bench.sh
  ls -la gpurun_out/*.ncu-rep; tail -3 gpurun_out/${TAG}_ncu_list.log
  for lib in libbsgpu.so libbsgpu_prev.so libbsgpu_r8.so; do
    echo "== $lib" >> gpurun_out/diag_async.log
    BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 120 python scripts/diag_async_stall.py 32 >> gpurun_out/diag_async.log 2>&1
  done
  cat gpurun_out/diag_async.log
  for lib in ${HALO_LIBS:-libbsgpu.so libbsgpu_ry2.so libbsgpu.so libbsgpu_ry2.so}; do
    BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 600 python bench.py --max-outer 30 --steps 20 --warmup 5 --no-cpu --no-config2 | tail -1 > gpurun_out/halo_ab_$lib.json
    python -c "import json; d=json.load(open('gpurun_out/halo_ab_$lib.json')); print('$lib config3 bounded', round(d['value'],2), 'Gpts/s', round(d['ms_per_step'],2), 'ms/step', round(d['roofline']['frac'],4), 'halo us', round(d['halo']['avg_us'],1), d['breakdown'])" | tee -a gpurun_out/halo_ab.log
  done
fi
