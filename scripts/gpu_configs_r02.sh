#!/bin/bash
# Every BASELINE model config through the default multi-GPU exchange at G = 2
# and 4 (scheduled exchange), plus the ResNet-269 chunk-size sweep at G = 4.
OUT=gpurun_out/$1; mkdir -p $OUT
run() { G=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
for cfg in resnet50 alexnet resnet269; do
  run 4 bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --config $cfg > $OUT/g4_$cfg.json 2>/dev/null
  CUDA_VISIBLE_DEVICES=0,1 run 2 bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --config $cfg \
      > $OUT/g2_$cfg.json 2>/dev/null
done
for cb in 4096 65536 1048576; do
  run 4 bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --config resnet269 --chunk-bytes $cb \
      > $OUT/g4_resnet269_cb$cb.json 2>/dev/null
done
echo done > $OUT/done
