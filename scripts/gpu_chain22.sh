# chain G = 2 on smaller models: block size vs pipeline fill.
mkdir -p gpurun_out/m22
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m22/build.log 2>&1
R="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --mode chain"
for cfg in resnet50 alexnet; do
  for b in 2048 4096 6144 8192; do $R --config $cfg --chain-block $b > gpurun_out/m22/${cfg}_b$b.json 2>/dev/null; done
done
for f in gpurun_out/m22/*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'])"; done
