#!/bin/bash
# Round-2 multi-GPU confirmation on 4 x B200 with the scheduled exchange as
# the default: driver-form bench lines at N = 4 and N = 2 (e2e included),
# the hierarchical line, NVLink counters of k_sched, the whole multi-GPU
# parity suite.   usage: bash scripts/gpu_multi_r02c.sh TAG
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
run() { G=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
run 4 bench.py --gpus 4 --steps 20 --warmup 5 > $OUT/bench_n4.json 2> $OUT/bench_n4.err
run 4 bench.py --gpus 4 --steps 20 --warmup 5 --mode hier --no-e2e > $OUT/bench_n4_hier.json 2> $OUT/bench_n4_hier.err
export CUDA_VISIBLE_DEVICES=0,1
run 2 bench.py --gpus 2 --steps 20 --warmup 5 > $OUT/bench_n2.json 2> $OUT/bench_n2.err
unset CUDA_VISIBLE_DEVICES
timeout 600 python scripts/nvlink_counters.py vgg19 sched > $OUT/nvl_plain.txt 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:"k_sched" --csv --log-file $OUT/nvl_ncu.csv \
    python scripts/nvlink_counters.py vgg19 sched > $OUT/nvl_ncu_stdout.txt 2>&1
timeout 3000 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider --timeout 900 \
    > $OUT/pytest_multi.txt 2>&1
echo done > $OUT/done
