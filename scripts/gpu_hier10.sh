# Round 1, session 2: hierarchical reduction (NEXT-4) parity + bench at G = 2, 4.
set -x
mkdir -p gpurun_out/m10
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m10/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "hier" > gpurun_out/m10/pytest_1gpu.log 2>&1; echo "pytest 1gpu $?"
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "hier or full_size" > gpurun_out/m10/pytest_multi.log 2>&1; echo "pytest multi $?"
for n in 2 4; do
  R="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 30 --warmup 5"
  $R --mode hier --no-e2e > gpurun_out/m10/n${n}_hier.json 2> gpurun_out/m10/n${n}_hier.err
  $R --mode hier --no-e2e --chain-block 32768 > gpurun_out/m10/n${n}_hier32k.json 2> gpurun_out/m10/n${n}_hier32k.err
  $R --no-e2e > gpurun_out/m10/n${n}_auto.json 2> gpurun_out/m10/n${n}_auto.err
done
for f in gpurun_out/m10/n*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'], d['scaling'], d['owner_phase']['value'])"; done
