#!/bin/bash
# Round-end style measurement: the driver's bench command (default config 3 at
# 512^3, full solve), the reference arm, then ncu evidence on a bounded run of
# the same command: the launch list (conditional CUDA graphs profiled as whole
# graphs: the per-sweep inner solve is one line, with its DRAM bytes) and one
# --set full capture of the sweep kernels in launch mode (BS_LAUNCH_MODE=1).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-r02}
if [ -z "$NO_BENCH" ]; then
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2> gpurun_out/${TAG}_bench.err
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.log 2>&1
fi
if [ -z "$NO_NCU" ]; then
ncu --graph-profiling graph --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --max-outer 8 --steps 3 --warmup 2 --no-cpu --no-config2 > gpurun_out/${TAG}_ncu_list.log 2>&1
BS_LAUNCH_MODE=1 ncu --set full --clock-control none --import-source on -k regex:k_sweep --launch-skip 400 -c 4 \
    -o gpurun_out/${TAG}_sweeps -f python bench.py --max-outer 4 --steps 1 --warmup 2 --no-cpu --no-config2 \
    > gpurun_out/${TAG}_ncu_full.log 2>&1
BS_LAUNCH_MODE=1 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 3 \
    -o gpurun_out/${TAG}_resid_jac -f python scripts/prof_jac.py 256 > gpurun_out/${TAG}_ncu_resid.log 2>&1
fi
