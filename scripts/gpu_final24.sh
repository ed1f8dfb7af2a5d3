# Last check of the committed state on 2 GPUs: smoke, default lines N = 1, 2, full GPU suite.
mkdir -p gpurun_out/m24
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m24/build.log 2>&1; echo "build $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m24/smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/m24/smoke.log
timeout 600 python bench.py > gpurun_out/m24/bench_n1.json 2> gpurun_out/m24/bench_n1.err; echo "n1 $?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/m24/bench_n2.json 2> gpurun_out/m24/bench_n2.err; echo "n2 $?"
for f in gpurun_out/m24/bench_*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'], (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('single_thread'))"; done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/m24/pytest_gpu_all.log 2>&1; echo "pytest all $?"; tail -2 gpurun_out/m24/pytest_gpu_all.log
