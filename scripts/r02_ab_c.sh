#!/bin/bash
# After the GIL switch-interval change: the async stall diagnostic (9 solves) and the async tests, three times
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for i in 1 2 3; do timeout 120 python scripts/diag_async_stall.py 32 >> gpurun_out/diag_async_v2.log 2>&1; done
cat gpurun_out/diag_async_v2.log
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_async_protocol.py tests/test_gpu_ipc.py -q -m gpu -p no:cacheprovider 2>&1 | tail -2 | tee -a gpurun_out/async_tests_v2.log; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "async" 2>&1 | tail -2 | tee -a gpurun_out/async_tests_v2.log
