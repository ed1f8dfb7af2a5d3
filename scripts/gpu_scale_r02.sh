#!/bin/bash
# Driver-form scaling preview on one 4-GPU box: N = 1, 2, 4 back to back with
# the defaults (python bench.py / torchrun ... bench.py --gpus N).
OUT=gpurun_out/$1; mkdir -p $OUT
python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/n1.json 2> $OUT/n1.err
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $N --steps 20 --warmup 5 \
      > $OUT/n$N.json 2> $OUT/n$N.err
done
echo done > $OUT/done
