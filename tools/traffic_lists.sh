#!/bin/bash
# ncu launch lists (DRAM bytes per kernel) of a short bench run per config,
# for profiles/ncu_traffic.json (the roofline's "traffic").
TAG=${1:-r05}
for c in c3 c4 c5; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/${TAG}_launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-graph --no-pnpn --no-gmres \
      --iters 5 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch_$c.log 2>&1
  echo "$c rc=$?"
done
