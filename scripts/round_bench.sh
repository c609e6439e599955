#!/bin/bash
# Round-end style measurement: the driver's bench command (default config 3 at
# 512^3, full solve), the reference arm, then ncu evidence on a bounded run of
# the same command (launch list + one --set full capture of the sweep kernels).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-r02}
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2> gpurun_out/${TAG}_bench.err
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${TAG}_ref.log 2>&1
if [ -z "$NO_NCU" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --max-outer 8 --steps 3 --warmup 2 --no-cpu --no-config2 > gpurun_out/${TAG}_ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep --launch-skip 400 -c 4 \
    -o gpurun_out/${TAG}_sweeps -f python bench.py --max-outer 4 --steps 1 --warmup 2 --no-cpu --no-config2 \
    > gpurun_out/${TAG}_ncu_full.log 2>&1
fi
