#!/bin/bash
# Scheduled exchange at G = 4 / 2: lag and block sweep, then the sched parity
# cases of tests/test_gpu_multi.py.   usage: bash scripts/gpu_sched_r02.sh TAG
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
run() { G=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
B="bench.py --steps 20 --warmup 5 --no-e2e"
for lag in 512 1024 2048 4096; do
  run 4 $B --gpus 4 --mode sched --sched-lag $lag > $OUT/g4_lag$lag.json 2> $OUT/g4_lag$lag.err
done
for blk in 8192 32768; do
  run 4 $B --gpus 4 --mode sched --sched-lag $((1024 * 16384 / blk)) --sched-block $blk \
      > $OUT/g4_blk$blk.json 2> $OUT/g4_blk$blk.err
done
export CUDA_VISIBLE_DEVICES=0,1
for lag in 0 64 256; do
  run 2 $B --gpus 2 --mode sched --sched-lag $lag > $OUT/g2_lag$lag.json 2> $OUT/g2_lag$lag.err
done
run 2 $B --gpus 2 --mode sched --sched-block 12288 > $OUT/g2_blk12288.json 2> $OUT/g2_blk12288.err
unset CUDA_VISIBLE_DEVICES
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider --timeout 600 -k sched \
    > $OUT/pytest_sched.txt 2>&1
echo done > $OUT/done
