# chain G = 2: producer / consumer grid sweep (CTA blocks of 16K).
mkdir -p gpurun_out/m18
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m18/build.log 2>&1
R="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --mode chain"
$R > gpurun_out/m18/base.json 2>/dev/null
for cg in 444 592 888; do $R --chain-consumer-grid $cg > gpurun_out/m18/cg$cg.json 2>/dev/null; done
for pg in 592 1184; do $R --chain-producer-grid $pg > gpurun_out/m18/pg$pg.json 2>/dev/null; done
$R --chain-producer-grid 1184 --chain-consumer-grid 592 > gpurun_out/m18/pg1184_cg592.json 2>/dev/null
$R --chain-block 12288 > gpurun_out/m18/b12k.json 2>/dev/null
$R --chain-block 20480 > gpurun_out/m18/b20k.json 2>/dev/null
for f in gpurun_out/m18/*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'])"; done
