#!/bin/bash
# Round-2 final single-GPU session on the final code: smoke, the whole GPU
# suite, the default bench line (driver form) + per-config lines + cache
# table + reference arm, ncu launch list and one --set full capture.
# usage: bash scripts/gpu_final_r02.sh TAG
OUT=gpurun_out/$1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > $OUT/pytest_gpu.txt 2>&1
python bench.py --steps 20 --warmup 5 > $OUT/bench_n1.json 2> $OUT/bench_n1.err
python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
python bench.py --steps 20 --warmup 5 --cache-table --no-cpu --no-e2e > $OUT/bench_cache_table.json 2>&1
for cfg in resnet50 alexnet resnet269 tiny; do
    python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu --no-e2e --graph > $OUT/bench_$cfg.json 2>&1
done
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    $CMD > $OUT/ncu_launch_stdout.txt 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_flat -s 3 -c 1 \
    -o $OUT/k_flat_vgg19 $CMD > $OUT/ncu_full_stdout.txt 2>&1
echo done > $OUT/done
