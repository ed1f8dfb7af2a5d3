# Start barriers restored: G = 2 parity (chain / push / hier) and the default N = 2 line.
mkdir -p gpurun_out/m27
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m27/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "(chain or push or hier or full_size) and not pull and not flags and not barrier and not warp and not window and not oneshot" > gpurun_out/m27/pytest_multi.log 2>&1; echo "pytest multi $?"; tail -1 gpurun_out/m27/pytest_multi.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/m27/bench_n2.json 2> gpurun_out/m27/bench_n2.err
grep -h '"value"' gpurun_out/m27/bench_n2.json | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('n2', d['value'], d['ms_per_step'], (d.get('e2e') or {}).get('value'))"
