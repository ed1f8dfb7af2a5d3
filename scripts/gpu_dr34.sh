# Double-buffered replicas (opt-in): push parity at G = 2 and the e2e effect.
mkdir -p gpurun_out/m34
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m34/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "push_dr and 2-" > gpurun_out/m34/pytest.log 2>&1; echo "pytest $?"; tail -1 gpurun_out/m34/pytest.log
R="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --mode push --e2e-steps 4"
$R > gpurun_out/m34/push.json 2>/dev/null
$R --double-replica > gpurun_out/m34/push_dr.json 2>/dev/null
for f in gpurun_out/m34/*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'])"; done
