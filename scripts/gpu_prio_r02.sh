#!/bin/bash
# kept-slice L2 priority (evict-last vs evict-normal) x size, bench-like setup,
# one fresh process per setting.   usage: bash scripts/gpu_prio_r02.sh TAG
# (the --resident-prio option was removed after this sweep: no gain, profiles/r02_prio/)
OUT=gpurun_out/$1; mkdir -p $OUT
B="python bench.py --steps 30 --warmup 10 --no-cpu --no-e2e"
for rep in 1 2; do
  $B --cache bypass > $OUT/bypass_$rep.json 2>&1
  for mb in 32 64 96 128; do
    for prio in 0 1; do
      $B --cache resident --resident-mb $mb --resident-prio $prio > $OUT/res_${mb}_p${prio}_$rep.json 2>&1
    done
  done
done
echo done > $OUT/done
