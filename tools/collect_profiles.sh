#!/bin/bash
# Run on the GPU box (under gpurun) from the repo root: the default bench
# line (c2, with the oracle CPU legs and the GMRES leg), the other configs,
# the affine variant, the DMMA probe, the full oracle CPU legs, the ncu launch
# list of a short bench command and one --set full capture of the CG kernels
# (stream order: ncu and conditional graph nodes are not mixed).  Outputs land
# in gpurun_out/.
TAG=${1:-r2}
python bench.py > gpurun_out/${TAG}_bench_c2.log 2>&1
for c in c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.log 2>&1
done
timeout 300 python bench.py --affine --steps 5 --no-cpu-baseline --no-gmres > gpurun_out/${TAG}_bench_c2_affine.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_probe tools/dmma_probe.cu && \
  timeout 120 tools/dmma_probe > gpurun_out/${TAG}_dmma_probe.log 2>&1
[ -n "$CPU_LEGS_ALL" ] && timeout 1500 python bench.py --cpu-legs all > gpurun_out/${TAG}_cpu_legs.json 2> gpurun_out/${TAG}_cpu_legs.err
CMD="python bench.py --steps 1 --warmup 3 --iters 5 --no-cpu-baseline --no-gmres --no-pnpn --no-graph"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
ITERS=3 python tools/prof_cg.py > gpurun_out/${TAG}_plain2.log 2>&1 && \
ITERS=3 ncu --set full --clock-control none --import-source on -k regex:"k_ax|k_gs_nodal|k_cg_update" \
    --launch-skip 1 -c 6 -o gpurun_out/${TAG}_full python tools/prof_cg.py > gpurun_out/${TAG}_ncu_full.log 2>&1
echo collected
