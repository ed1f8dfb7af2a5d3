# Round 1, session 2: M3 push exchange (all-store owner-sharded) vs P2P at G = 2, 4.
set -x
mkdir -p gpurun_out/m14
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m14/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "push or hier" > gpurun_out/m14/pytest_multi.log 2>&1; echo "pytest multi $?"; tail -2 gpurun_out/m14/pytest_multi.log
for n in 4 2; do
  R="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 30 --warmup 5 --no-e2e"
  for b in 16384 32768 65536; do
    $R --mode push --hier-block $b > gpurun_out/m14/n${n}_push_b$b.json 2> gpurun_out/m14/n${n}_push_b$b.err
  done
  $R --mode p2p > gpurun_out/m14/n${n}_p2p.json 2> gpurun_out/m14/n${n}_p2p.err
done
for f in gpurun_out/m14/n*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'], d['roofline_nvlink']['frac'])"; done
