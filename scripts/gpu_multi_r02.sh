#!/bin/bash
# Round-2 multi-GPU session (gpurun --gpus G): parity tests, bench lines, NVLink counters.
# usage: bash scripts/gpu_multi_r02.sh G TAG
G=$1; TAG=$2; OUT=gpurun_out/$TAG; mkdir -p $OUT
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
CUDA_VISIBLE_DEVICES=0 ./scripts/cache_sweep > $OUT/cache_sweep.jsonl 2>&1
timeout 2400 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider --timeout 900 \
    > $OUT/pytest_multi.txt 2>&1
for mode in auto push hier allreduce nccl p2p; do
    run bench.py --gpus $G --steps 20 --warmup 5 --mode $mode > $OUT/bench_$mode.json 2> $OUT/bench_$mode.err
done
run bench.py --gpus $G --steps 20 --warmup 5 --mode push --workers $((8 * G)) --no-e2e \
    > $OUT/bench_push_flat$((8 * G)).json 2> $OUT/bench_push_flat.err
timeout 600 python scripts/nvlink_counters.py vgg19 > $OUT/nvl_plain.txt 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:"k_hier|k_blocks|k_flat" --csv --log-file $OUT/nvl_ncu.csv \
    python scripts/nvlink_counters.py vgg19 > $OUT/nvl_ncu_stdout.txt 2>&1
echo done > $OUT/done
