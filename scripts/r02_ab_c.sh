#!/bin/bash
# After the GIL switch-interval change: the async stall diagnostic (9 solves) and the async tests, three times
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for i in 1 2 3; do timeout 120 python scripts/diag_async_stall.py 32 >> gpurun_out/diag_async_v2.log 2>&1; done
cat gpurun_out/diag_async_v2.log
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_async_protocol.py tests/test_gpu_ipc.py -q -m gpu -p no:cacheprovider 2>&1 | tail -2 | tee -a gpurun_out/async_tests_v2.log; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "async" 2>&1 | tail -2 | tee -a gpurun_out/async_tests_v2.log
# bitwise-neutral ring variants on the bounded config-3 bench: S1 plane pairs, 9-plane S1 ring, 14-plane S2 ring
for lib in libbsgpu.so libbsgpu_zps1.so libbsgpu_ab9.so libbsgpu_a14.so libbsgpu.so; do
  BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 600 python bench.py --max-outer 30 --steps 20 --warmup 5 --no-cpu --no-config2 | tail -1 > gpurun_out/ring_ab_$lib.json
  python -c "import json; d=json.load(open('gpurun_out/ring_ab_$lib.json')); print('$lib config3 bounded', round(d['value'],2), 'Gpts/s', round(d['ms_per_step'],2), 'ms/step', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])" | tee -a gpurun_out/ring_ab.log
done
