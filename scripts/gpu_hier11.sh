# Round 1, session 2: k_hier at 3 CTAs/SM (batched loads), block sweep; full GPU suite.
set -x
mkdir -p gpurun_out/m11
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m11/build.log 2>&1
for n in 2 4; do
  for b in 32768 65536 131072; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 30 --warmup 5 --mode hier --no-e2e --hier-block $b > gpurun_out/m11/n${n}_hier_b$b.json 2> gpurun_out/m11/n${n}_hier_b$b.err
  done
done
for f in gpurun_out/m11/n*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'], d['roofline_nvlink']['frac'])"; done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/m11/pytest_gpu_all.log 2>&1; echo "pytest all $?"; tail -3 gpurun_out/m11/pytest_gpu_all.log
