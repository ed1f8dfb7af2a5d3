# Start barriers restored: the default N = 4 line and G = 4 push / hier parity.
mkdir -p gpurun_out/m28
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m28/build.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 > gpurun_out/m28/bench_n4.json 2> gpurun_out/m28/bench_n4.err
grep -h '"value"' gpurun_out/m28/bench_n4.json | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('n4', d['value'], d['ms_per_step'], (d.get('e2e') or {}).get('value'))"
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "(push or hier) and not vgg19 and not 2-" > gpurun_out/m28/pytest_multi.log 2>&1; echo "pytest multi $?"; tail -1 gpurun_out/m28/pytest_multi.log
