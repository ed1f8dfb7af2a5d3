#!/bin/bash
OUT=gpurun_out/l2_hint.jsonl; : > $OUT
./scripts/l2_hint 0 0 0 >> $OUT 2>&1
for mb in 32 64 96; do for lk in 0 1 2; do for sk in 0 1 2; do ./scripts/l2_hint $mb $lk $sk >> $OUT 2>&1; done; done; done
./scripts/l2_hint 0 0 0 >> $OUT 2>&1
