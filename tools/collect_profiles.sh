#!/bin/bash
# Run on the GPU box (under gpurun) from the repo root: the default bench
# line, the other configs, the ncu launch list of a short bench command and
# one --set full capture of the CG kernels.  Outputs land in gpurun_out/.
set -e
TAG=${1:-r06}
python bench.py > gpurun_out/${TAG}_bench_c2.log 2>&1
for c in c3 c4 c5; do
  python bench.py --config $c --steps 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.log 2>&1
done
CMD="python bench.py --steps 1 --warmup 3 --iters 5 --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
ITERS=3 python tools/prof_cg.py > gpurun_out/${TAG}_plain2.log 2>&1
ITERS=3 ncu --set full --clock-control none --import-source on -k regex:"k_ax|k_gs_nodal|k_cg_update" \
    --launch-skip 1 -c 6 -o gpurun_out/${TAG}_full python tools/prof_cg.py > gpurun_out/${TAG}_ncu_full.log 2>&1
echo collected
