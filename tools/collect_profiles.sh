#!/bin/bash
# Run on the GPU box (under gpurun) from the repo root: plain bench, then the
# ncu launch list of a short bench command and one --set full capture of the
# fused CG operator kernel.  Outputs land in gpurun_out/.
set -e
TAG=${1:-r01}
CMD="python bench.py --steps 1 --warmup 3 --iters 5 --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
python tools/prof_ax.py > gpurun_out/${TAG}_plain2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_ax|k_gs_flat|k_cg_update" -c 8 \
    -o gpurun_out/${TAG}_full python tools/prof_ax.py > gpurun_out/${TAG}_ncu_full.log 2>&1
echo collected
