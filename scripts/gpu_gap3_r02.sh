#!/bin/bash
# C vs Python-without-torch vs Python-with-torch vs bench, fresh process each
OUT=gpurun_out/r02_gap3; mkdir -p $OUT
for rep in 1 2 3; do
  for cache in 1 2; do
    ./scripts/flat_c_probe $cache
    python scripts/flat_py_probe.py notorch $cache
    python scripts/flat_py_probe.py torch $cache
  done
  ./scripts/flat_variants r | grep '"pass": 2' | head -1
done > $OUT/out.jsonl 2>&1
cat $OUT/out.jsonl
