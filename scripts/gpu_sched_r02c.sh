#!/bin/bash
# Scheduled exchange with producer / consumer lanes: G = 4 / 2 sweep, the
# emulated-rank tests on GPU 0, and the sched parity cases at G = 2, 4.
# usage: bash scripts/gpu_sched_r02c.sh TAG
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
run() { G=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
B="bench.py --steps 20 --warmup 5 --no-e2e"
run 4 $B --gpus 4 --mode auto > $OUT/g4_push.json 2> $OUT/g4_push.err
for lag in 0 256 1024; do
  run 4 $B --gpus 4 --mode sched --sched-lag $lag > $OUT/g4_lag$lag.json 2> $OUT/g4_lag$lag.err
done
for cons in 64 148 222; do
  run 4 $B --gpus 4 --mode sched --sched-consumers $cons > $OUT/g4_cons$cons.json 2> $OUT/g4_cons$cons.err
done
run 4 $B --gpus 4 --mode sched --sched-block 32768 > $OUT/g4_blk32768.json 2> $OUT/g4_blk32768.err
run 4 $B --gpus 4 --mode sched --sched-weights 0.125,0.25,0.25,0.375 --sched-raw 1,0,0,0 \
    > $OUT/g4_hybrid.json 2> $OUT/g4_hybrid.err
export CUDA_VISIBLE_DEVICES=0,1
run 2 $B --gpus 2 --mode auto > $OUT/g2_chain.json 2> $OUT/g2_chain.err
run 2 $B --gpus 2 --mode sched > $OUT/g2_sched.json 2> $OUT/g2_sched.err
export CUDA_VISIBLE_DEVICES=0
timeout 600 python -m pytest tests/test_gpu_emulated_ranks.py -q -p no:cacheprovider --timeout 300 \
    -k sched > $OUT/pytest_emulated.txt 2>&1
unset CUDA_VISIBLE_DEVICES
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider --timeout 600 -k sched \
    > $OUT/pytest_sched.txt 2>&1
echo done > $OUT/done
