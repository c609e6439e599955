#!/bin/bash
# Async driver with the receive after the posts (reference order): stall scenario, delay staleness, async tests
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for i in 1 2 3 4 5; do timeout 120 python scripts/diag_async_stall.py 32 >> gpurun_out/diag_async_v5.log 2>&1; done
cat gpurun_out/diag_async_v5.log
timeout 300 python scripts/diag_async_delay.py > gpurun_out/diag_async_delay.log 2>&1; cat gpurun_out/diag_async_delay.log
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_async_protocol.py tests/test_gpu_ipc.py tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "async or ipc or suspended or ring or torn" 2>&1 | tail -8 | tee -a gpurun_out/async_tests_v3.log; done
timeout 1100 python scripts/cfg4_bar.py > gpurun_out/cfg4_bar_v2.log 2>&1; tail -3 gpurun_out/cfg4_bar_v2.log
