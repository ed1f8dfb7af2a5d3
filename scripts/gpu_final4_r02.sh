#!/bin/bash
# Round-2 final multi-GPU session on 4 x B200 with the final code: driver-form
# bench lines at N = 4 and N = 2, the whole multi-GPU parity suite, and one
# ncu --set full capture of k_sched (rank 0, flags pre-raised).
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
run() { G=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
run 4 bench.py --gpus 4 --steps 20 --warmup 5 > $OUT/bench_n4.json 2> $OUT/bench_n4.err
export CUDA_VISIBLE_DEVICES=0,1
run 2 bench.py --gpus 2 --steps 20 --warmup 5 > $OUT/bench_n2.json 2> $OUT/bench_n2.err
unset CUDA_VISIBLE_DEVICES
timeout 600 python scripts/nvlink_counters.py vgg19 sched > $OUT/nvl_plain.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sched -c 1 \
    -o $OUT/k_sched_g4 python scripts/nvlink_counters.py vgg19 sched > $OUT/ncu_full_stdout.txt 2>&1
timeout 3000 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider --timeout 900 \
    > $OUT/pytest_multi.txt 2>&1
echo done > $OUT/done
