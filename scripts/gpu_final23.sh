# chain without the start barrier; push block sweep at G = 4.
mkdir -p gpurun_out/m23
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m23/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "chain or full_size" > gpurun_out/m23/pytest_multi.log 2>&1; echo "pytest multi $?"; tail -1 gpurun_out/m23/pytest_multi.log
R2="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2"
R4="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4"
$R2 > gpurun_out/m23/bench_n2.json 2> gpurun_out/m23/bench_n2.err
$R2 --config resnet50 --no-e2e > gpurun_out/m23/rn50_n2.json 2>/dev/null
for b in 8192 12288 16384; do $R4 --no-e2e --push-block $b > gpurun_out/m23/push_b$b.json 2>/dev/null; done
for f in gpurun_out/m23/*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'], (d.get('e2e') or {}).get('value'))"; done
