# Round 1, session 2: block-streaming chain with dynamic block tickets.
set -x
mkdir -p gpurun_out/m9
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m9/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "block_streaming or consume or stage_flags or chain" > gpurun_out/m9/pytest_1gpu.log 2>&1; echo "pytest 1gpu $?"
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "chain" > gpurun_out/m9/pytest_multi.log 2>&1; echo "pytest multi $?"
R="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --mode chain"
for rep in 1 2; do
for b in 8192 16384 32768 65536; do
  $R --chain-block $b > gpurun_out/m9/n2_b${b}_r$rep.json 2> gpurun_out/m9/n2_b${b}_r$rep.err
  $R --chain-block $b --chain-producer-grid 296 > gpurun_out/m9/n2_b${b}_pg296_r$rep.json 2> gpurun_out/m9/n2_b${b}_pg296_r$rep.err
done
done
for f in gpurun_out/m9/n2_*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'], d['owner_phase'])"; done
