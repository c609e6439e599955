#!/bin/bash
# Round-2 check before the segmented config-5 run: new tests, a small segmented dry run of
# scripts/run_cfg5.py (pause / resume through /tmp), and the library A/B of the lean residual / Jacobi rounds.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_checkpoint.py tests/test_gpu_parity.py tests/test_gpu_persistent.py -x -q -m gpu > gpurun_out/check_a_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/check_a_pytest.log
tail -3 gpurun_out/check_a_pytest.log
# dry run: 256^3 in segments of ~14 s, against one uninterrupted run
rm -rf /tmp/cfg5_dry
CKPT_DIR=/tmp/cfg5_dry LOG_EVERY=50 timeout 600 python scripts/run_cfg5.py 256 > gpurun_out/check_a_dry_full.log 2>&1
R=0
for s in 1 2 3 4 5 6 7 8; do
  RESUME=$R SEG_BUDGET_S=14 CKPT_DIR=/tmp/cfg5_dry LOG_EVERY=50 timeout 600 python scripts/run_cfg5.py 256 > gpurun_out/check_a_dry_seg$s.log 2>&1
  R=1
  if grep -q '"done"' gpurun_out/check_a_dry_seg$s.log; then break; fi
done
tail -1 gpurun_out/check_a_dry_full.log; tail -1 gpurun_out/check_a_dry_seg$s.log
LIBS="libbsgpu_prev.so libbsgpu.so libbsgpu_r10.so libbsgpu_r12j16.so libbsgpu_r12j20.so" NOBENCH=1 bash scripts/lib_sweeps_ab.sh > gpurun_out/check_a_ab.log 2>&1
cat gpurun_out/check_a_ab.log
