#!/bin/bash
# Multi-GPU bench lines (run under gpurun --gpus 4): c2 weak and c3 strong
# scaling at 2 and 4 GPUs; logs in gpurun_out/<tag>_scale_<cfg>_<n>.log
TAG=${1:-r05}
for n in 2 4; do for c in c2 c3; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2951$n bench.py --gpus $n --config $c --steps 10 --warmup 3 > gpurun_out/${TAG}_scale_${c}_$n.log 2>&1
  echo "n=$n $c rc=$?"
done; done
