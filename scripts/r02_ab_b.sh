#!/bin/bash
# Ring-depth A/B of the lean residual / Jacobi sweeps, then ncu evidence of the serving sweeps at 256^3
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
LIBS="libbsgpu.so libbsgpu_mixed.so libbsgpu_r14j10.so libbsgpu_r16j8.so" NOBENCH=1 SLAB=1 bash scripts/lib_sweeps_ab.sh > gpurun_out/ab_b.log 2>&1
cat gpurun_out/ab_b.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sweep -c 8 -o gpurun_out/r02_lean_sweeps -f \
  python scripts/prof_jac.py 256 > gpurun_out/ab_b_ncu.log 2>&1
ls -la gpurun_out/*.ncu-rep
for lib in libbsgpu.so libbsgpu_mixed.so libbsgpu.so libbsgpu_mixed.so; do
  BS_LIB=$PWD/paper_2009_12638_b200/_lib/$lib timeout 600 python bench.py --max-outer 30 --steps 20 --warmup 5 --no-cpu --no-config2 | tail -1 > gpurun_out/ab_b_bench_$lib.json
  python -c "import json; d=json.load(open('gpurun_out/ab_b_bench_$lib.json')); print('$lib config3 bounded', round(d['value'],2), 'Gpts/s', round(d['ms_per_step'],2), 'ms/step', round(d['roofline']['frac'],4), 'halo us', round(d['halo']['avg_us'],1))" | tee -a gpurun_out/ab_b.log
done
BS_LIB=$PWD/paper_2009_12638_b200/_lib/libbsgpu_mixed.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_persistent.py tests/test_gpu_placement.py -x -q -m gpu 2>&1 | tail -2 | tee -a gpurun_out/ab_b.log
