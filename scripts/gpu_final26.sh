# N = 4 default line (push exchange, 12K blocks) and hierarchical G = 4 with the final code.
mkdir -p gpurun_out/m26
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m26/build.log 2>&1
R4="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4"
$R4 > gpurun_out/m26/bench_n4.json 2> gpurun_out/m26/bench_n4.err
$R4 --mode hier --no-e2e > gpurun_out/m26/hier_n4.json 2>/dev/null
for f in gpurun_out/m26/*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'], (d.get('e2e') or {}).get('value'), d['roofline_nvlink'].get('frac'))"; done
