# Round 1, session 2: chain with CONSUME (L2 discard of the inbox), producer grid, block sizes.
set -x
mkdir -p gpurun_out/m8
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m8/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "block_streaming or consume or stage_flags or chain" > gpurun_out/m8/pytest_1gpu.log 2>&1; echo "pytest 1gpu $?"
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "chain" > gpurun_out/m8/pytest_multi.log 2>&1; echo "pytest multi $?"
R="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --mode chain"
for b in 16384 24576 32768; do
  $R --chain-block $b > gpurun_out/m8/n2_b${b}.json 2> gpurun_out/m8/n2_b${b}.err
  $R --chain-block $b --chain-no-consume > gpurun_out/m8/n2_b${b}_noconsume.json 2> gpurun_out/m8/n2_b${b}_noconsume.err
  $R --chain-block $b --chain-producer-grid 296 > gpurun_out/m8/n2_b${b}_pg296.json 2> gpurun_out/m8/n2_b${b}_pg296.err
  $R --chain-block $b --chain-producer-grid 148 > gpurun_out/m8/n2_b${b}_pg148.json 2> gpurun_out/m8/n2_b${b}_pg148.err
done
$R --chain-block 8192 --chain-producer-grid 296 > gpurun_out/m8/n2_b8192_pg296.json 2> gpurun_out/m8/n2_b8192_pg296.err
for f in gpurun_out/m8/n2_*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'])"; done
