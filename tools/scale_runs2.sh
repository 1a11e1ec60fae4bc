#!/bin/bash
# c4 (weak, 48^3 per GPU) and c5 (strong, cylinder lx10) at 2 and 4 GPUs
TAG=${1:-r06}
for n in 2 4; do for c in c4 c5; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2952$n bench.py --gpus $n --config $c --steps 5 --warmup 3 > gpurun_out/${TAG}_scale_${c}_$n.log 2>&1
  echo "n=$n $c rc=$?"
done; done
