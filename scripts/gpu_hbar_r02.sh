#!/bin/bash
# k_hier with in-kernel round barriers: emulated tests on GPU 0, hier / push
# bench lines at G = 4 and 2, multi-GPU hier / push parity.   usage: ... TAG
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
run() { G=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
export CUDA_VISIBLE_DEVICES=0
timeout 1200 python -m pytest tests/test_gpu_emulated_ranks.py -q -p no:cacheprovider --timeout 300 \
    > $OUT/pytest_emulated.txt 2>&1
unset CUDA_VISIBLE_DEVICES
B="bench.py --steps 30 --warmup 5 --no-e2e"
for rep in 1 2; do
  run 4 $B --gpus 4 --mode hier > $OUT/g4_hier_$rep.json 2>/dev/null
  run 4 $B --gpus 4 --mode push > $OUT/g4_push_$rep.json 2>/dev/null
done
export CUDA_VISIBLE_DEVICES=0,1
run 2 $B --gpus 2 --mode hier > $OUT/g2_hier.json 2>/dev/null
unset CUDA_VISIBLE_DEVICES
timeout 2400 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider --timeout 900 \
    -k "hier or push or auto" > $OUT/pytest_multi.txt 2>&1
echo done > $OUT/done
