#!/bin/bash
# Pipeline taper sweep at G = 4 and G = 2 + emulated sched parity on GPU 0.
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
run() { G=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
B="bench.py --steps 30 --warmup 5 --no-e2e --mode sched"
for rep in 1 2; do
  for tp in 0 8 32 128; do
    run 4 $B --gpus 4 --sched-taper $tp > $OUT/g4_taper${tp}_$rep.json 2>/dev/null
  done
done
export CUDA_VISIBLE_DEVICES=0,1
for tp in 0 8 32; do
  run 2 $B --gpus 2 --sched-taper $tp > $OUT/g2_taper$tp.json 2>/dev/null
done
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_emulated_ranks.py -q -p no:cacheprovider --timeout 300 -k sched \
    > $OUT/pytest_emulated.txt 2>&1
echo done > $OUT/done
