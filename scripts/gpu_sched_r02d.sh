#!/bin/bash
# Interleaved scheduled exchange: G = 4 lag / block / consumer sweep, G = 2
# chain vs sched alternated, sched parity (emulated on GPU 0 + G = 2, 4).
# usage: bash scripts/gpu_sched_r02d.sh TAG
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
run() { G=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
B="bench.py --steps 30 --warmup 5 --no-e2e"
for rep in 1 2; do
  run 4 $B --gpus 4 --mode push > $OUT/g4_push_$rep.json 2>/dev/null
  run 4 $B --gpus 4 --mode sched > $OUT/g4_sched_$rep.json 2>/dev/null
done
for lag in 64 256 1024; do
  run 4 $B --gpus 4 --mode sched --sched-lag $lag > $OUT/g4_lag$lag.json 2>/dev/null
done
for blk in 8192 12288 24576; do
  run 4 $B --gpus 4 --mode sched --sched-block $blk > $OUT/g4_blk$blk.json 2>/dev/null
done
for cons in 96 160; do
  run 4 $B --gpus 4 --mode sched --sched-consumers $cons > $OUT/g4_cons$cons.json 2>/dev/null
done
run 4 $B --gpus 4 --mode sched --sched-weights 0.125,0.25,0.25,0.375 --sched-raw 1,0,0,0 \
    > $OUT/g4_hybrid.json 2>/dev/null
run 4 $B --gpus 4 --mode sched --sched-weights 0.25,0.25,0.25,0.25 --sched-raw 1,1,1,1 \
    > $OUT/g4_allraw.json 2>/dev/null
export CUDA_VISIBLE_DEVICES=0,1
for rep in 1 2 3; do
  run 2 $B --gpus 2 --mode chain > $OUT/g2_chain_$rep.json 2>/dev/null
  run 2 $B --gpus 2 --mode sched > $OUT/g2_sched_$rep.json 2>/dev/null
done
run 2 $B --gpus 2 --mode sched --sched-block 32768 > $OUT/g2_blk32768.json 2>/dev/null
run 2 $B --gpus 2 --mode sched --sched-block 8192 > $OUT/g2_blk8192.json 2>/dev/null
export CUDA_VISIBLE_DEVICES=0
timeout 600 python -m pytest tests/test_gpu_emulated_ranks.py -q -p no:cacheprovider --timeout 300 \
    -k sched > $OUT/pytest_emulated.txt 2>&1
unset CUDA_VISIBLE_DEVICES
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider --timeout 600 -k sched \
    > $OUT/pytest_sched.txt 2>&1
echo done > $OUT/done
