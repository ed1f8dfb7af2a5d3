# Round 1, session 2: round-end rehearsal -- build, smoke, default bench lines at N = 1, 2, 4
# (driver launch form, e2e included), reference arm, full GPU suite.
set -x
mkdir -p gpurun_out/m15
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m15/build.log 2>&1; echo "build $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m15/smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/m15/smoke.log
timeout 600 python bench.py > gpurun_out/m15/bench_n1.json 2> gpurun_out/m15/bench_n1.err; echo "n1 $?"
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n > gpurun_out/m15/bench_n$n.json 2> gpurun_out/m15/bench_n$n.err; echo "n$n $?"
done
timeout 600 python bench.py --impl reference > gpurun_out/m15/bench_ref.json 2> gpurun_out/m15/bench_ref.err; echo "ref $?"
for f in gpurun_out/m15/bench_*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'], (d.get('e2e') or {}).get('value'), d['config'].get('mode','')[:40])"; done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/m15/pytest_gpu_all.log 2>&1; echo "pytest all $?"; tail -3 gpurun_out/m15/pytest_gpu_all.log
