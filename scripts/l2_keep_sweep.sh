#!/bin/bash
# one fresh process per configuration (L2 state must not carry over between configs)
OUT=gpurun_out/l2_keep.jsonl; : > $OUT
for cfg in "0 0" "16 0" "32 0" "48 0" "64 0" "80 0" "96 0" "112 0" "0 32" "0 64" "0 96" "24 24" "32 32" "48 48" "64 64" "0 0"; do
    ./scripts/l2_keep $cfg >> $OUT 2>&1
done
