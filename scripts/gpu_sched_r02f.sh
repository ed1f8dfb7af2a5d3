#!/bin/bash
# Owner shares from the LP with per-stage capacity discounts (the chain's later
# stages start later): eps = 0 / 0.02 / 0.03, two repetitions, G = 4.
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
run() { G=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) "$@"; }
B="bench.py --gpus 4 --steps 30 --warmup 5 --no-e2e --mode sched"
for rep in 1 2; do
  run 4 $B > $OUT/eps0_$rep.json 2>/dev/null
  run 4 $B --sched-weights 0.3258,0.2044,0.1871,0.2827 --sched-raw 0.5247,0.0363,0,0.1448 > $OUT/eps2_$rep.json 2>/dev/null
  run 4 $B --sched-weights 0.3404,0.2105,0.184,0.2651 --sched-raw 0.5226,0.0539,0,0.131 > $OUT/eps3_$rep.json 2>/dev/null
done
echo done > $OUT/done
