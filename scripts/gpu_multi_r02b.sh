#!/bin/bash
# Round-2 multi-GPU session b (gpurun --gpus 4): multi-GPU parity incl. the
# scheduled exchange, then bench lines at G = 4 and G = 2 (push / chain /
# sched variants / hier).   usage: bash scripts/gpu_multi_r02b.sh TAG
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
run() { G=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
B="bench.py --steps 20 --warmup 5 --no-e2e"
run 4 $B --gpus 4 --mode auto > $OUT/g4_auto.json 2> $OUT/g4_auto.err
run 4 $B --gpus 4 --mode sched > $OUT/g4_sched.json 2> $OUT/g4_sched.err
for lag in 64 256; do
  run 4 $B --gpus 4 --mode sched --sched-lag $lag > $OUT/g4_sched_lag$lag.json 2> $OUT/g4_sched_lag$lag.err
done
for blk in 8192 32768; do
  run 4 $B --gpus 4 --mode sched --sched-block $blk > $OUT/g4_sched_blk$blk.json 2> $OUT/g4_sched_blk$blk.err
done
run 4 $B --gpus 4 --mode sched --sched-weights 0.125,0.25,0.25,0.375 --sched-raw 1,0,0,0 \
    > $OUT/g4_sched_hybrid.json 2> $OUT/g4_sched_hybrid.err
export CUDA_VISIBLE_DEVICES=0,1
run 2 $B --gpus 2 --mode auto > $OUT/g2_auto.json 2> $OUT/g2_auto.err
run 2 $B --gpus 2 --mode sched > $OUT/g2_sched.json 2> $OUT/g2_sched.err
unset CUDA_VISIBLE_DEVICES
timeout 3000 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider --timeout 900 \
    > $OUT/pytest_multi.txt 2>&1
echo done > $OUT/done
