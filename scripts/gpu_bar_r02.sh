#!/bin/bash
# In-kernel round barriers of the scheduled exchange vs NCCL barriers, 4 x B200:
# emulated-rank sched tests on GPU 0, bench lines at G = 4 and G = 2 (both
# barrier kinds, alternated), the sched multi-GPU parity cases.
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
run() { G=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests/test_gpu_emulated_ranks.py -q -p no:cacheprovider --timeout 300 -k sched \
    > $OUT/pytest_emulated.txt 2>&1
unset CUDA_VISIBLE_DEVICES
B="bench.py --steps 30 --warmup 5"
for rep in 1 2; do
  run 4 $B --gpus 4 --no-e2e > $OUT/g4_dev_$rep.json 2> $OUT/g4_dev_$rep.err
  run 4 $B --gpus 4 --no-e2e --sched-host-barrier > $OUT/g4_host_$rep.json 2>/dev/null
done
export CUDA_VISIBLE_DEVICES=0,1
for rep in 1 2; do
  run 2 $B --gpus 2 --no-e2e > $OUT/g2_dev_$rep.json 2> $OUT/g2_dev_$rep.err
  run 2 $B --gpus 2 --no-e2e --sched-host-barrier > $OUT/g2_host_$rep.json 2>/dev/null
done
unset CUDA_VISIBLE_DEVICES
run 4 $B --gpus 4 > $OUT/g4_dev_e2e.json 2> $OUT/g4_dev_e2e.err
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider --timeout 600 -k "sched or auto" \
    > $OUT/pytest_multi.txt 2>&1
echo done > $OUT/done
