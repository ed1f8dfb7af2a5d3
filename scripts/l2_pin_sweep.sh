#!/bin/bash
# one fresh process per configuration
OUT=gpurun_out/l2_pin.jsonl; : > $OUT
./scripts/l2_pin 0 0 1 4 >> $OUT 2>&1
for mb in 16 32 64 96 128; do ./scripts/l2_pin $mb 0 1 4 >> $OUT 2>&1; done
for mb in 32 64; do ./scripts/l2_pin 0 $mb 1 4 >> $OUT 2>&1; done
./scripts/l2_pin 32 32 1 4 >> $OUT 2>&1
./scripts/l2_pin 64 64 1 4 >> $OUT 2>&1
for mb in 32 64; do ./scripts/l2_pin $mb 0 2 4 >> $OUT 2>&1; done
./scripts/l2_pin 64 0 1 40 >> $OUT 2>&1
./scripts/l2_pin 0 0 1 4 >> $OUT 2>&1
