#!/bin/bash
# fresh process per setting (the L2 state a run leaves carries over)
OUT=gpurun_out/r02_gap; mkdir -p $OUT
for rep in 1 2; do
  for alloc in torch cuda; do
    for ple in 0 1; do
      for cache in 1 2; do
        python scripts/flat_gap_probe.py $alloc $ple $cache >> $OUT/gap.jsonl 2>> $OUT/err.txt
      done
    done
  done
done
./scripts/flat_variants r > $OUT/standalone.jsonl 2>&1
cat $OUT/gap.jsonl
