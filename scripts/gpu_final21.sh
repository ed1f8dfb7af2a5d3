# Round 1 session 2 final: configs x G table (auto exchange), RN269 chunk sweep at G = 4,
# default lines N = 1, 2, 4, smoke, full GPU suite.
set -x
mkdir -p gpurun_out/m21
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m21/build.log 2>&1; echo "build $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m21/smoke.log 2>&1; echo "smoke $?"
timeout 600 python bench.py > gpurun_out/m21/bench_n1.json 2> gpurun_out/m21/bench_n1.err; echo "n1 $?"
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n > gpurun_out/m21/bench_n$n.json 2> gpurun_out/m21/bench_n$n.err; echo "n$n $?"
done
for cfg in resnet50 alexnet resnet269; do
  timeout 300 python bench.py --config $cfg --no-e2e --no-cpu > gpurun_out/m21/cfg_${cfg}_n1.json 2>/dev/null
  for n in 2 4; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --config $cfg --no-e2e > gpurun_out/m21/cfg_${cfg}_n$n.json 2>/dev/null
  done
done
for cb in 4096 32768 262144 1048576; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --config resnet269 --chunk-bytes $cb --no-e2e > gpurun_out/m21/rn269_cb${cb}_n4.json 2>/dev/null
done
for f in gpurun_out/m21/*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'], (d.get('e2e') or {}).get('value'))"; done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/m21/pytest_gpu_all.log 2>&1; echo "pytest all $?"; tail -3 gpurun_out/m21/pytest_gpu_all.log
