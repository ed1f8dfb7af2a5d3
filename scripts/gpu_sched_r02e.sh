#!/bin/bash
# RAW_PUSH unrolled 4/W vectors per thread: G = 4 default / all-RAW vs push,
# emulated-rank parity on GPU 0.   usage: bash scripts/gpu_sched_r02e.sh TAG
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
run() { G=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
B="bench.py --steps 30 --warmup 5 --no-e2e"
for rep in 1 2; do
  run 4 $B --gpus 4 > $OUT/g4_auto_$rep.json 2>/dev/null
  run 4 $B --gpus 4 --mode push > $OUT/g4_push_$rep.json 2>/dev/null
  run 4 $B --gpus 4 --mode sched --sched-weights 0.25,0.25,0.25,0.25 --sched-raw 1,1,1,1 \
      > $OUT/g4_allraw_$rep.json 2>/dev/null
done
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_emulated_ranks.py -q -p no:cacheprovider --timeout 300 \
    > $OUT/pytest_emulated.txt 2>&1
echo done > $OUT/done
