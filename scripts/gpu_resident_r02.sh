#!/bin/bash
# Round-2 L2-resident slice sweep with the policy-operand kernel (44 registers):
# one fresh process per setting (the L2 state a run leaves matters,
# profiles/r02_l2/), then the cache-policy parity tests and one ncu capture.
# usage: bash scripts/gpu_resident_r02.sh TAG
OUT=gpurun_out/$1; mkdir -p $OUT
B="python bench.py --steps 30 --warmup 10 --no-cpu --no-e2e"
for rep in 1 2; do
  $B --cache bypass > $OUT/bypass_$rep.json 2>&1
  for mb in 0 16 32 48 64 96 128; do
    $B --cache resident --resident-mb $mb > $OUT/resident_${mb}_$rep.json 2>&1
  done
done
timeout 900 python -m pytest tests/test_gpu_order.py tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 > $OUT/pytest.txt 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    $CMD > $OUT/ncu_launch_stdout.txt 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_flat -s 3 -c 1 \
    -o $OUT/k_flat_vgg19 $CMD > $OUT/ncu_full_stdout.txt 2>&1
echo done > $OUT/done
