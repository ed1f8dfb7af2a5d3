# Round 1, session 2: warp-granular block streaming for the chain.
set -x
mkdir -p gpurun_out/m17
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m17/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "block_streaming or chain or hier" > gpurun_out/m17/pytest_1gpu.log 2>&1; echo "pytest 1gpu $?"; tail -1 gpurun_out/m17/pytest_1gpu.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "chain and bit_exact" > gpurun_out/m17/pytest_multi.log 2>&1; echo "pytest multi $?"; tail -1 gpurun_out/m17/pytest_multi.log
R="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --mode chain"
$R > gpurun_out/m17/n2_base.json 2> gpurun_out/m17/n2_base.err
for b in 1024 2048 4096 8192; do
  $R --chain-per-warp --chain-block $b > gpurun_out/m17/n2_w_b$b.json 2> gpurun_out/m17/n2_w_b$b.err
  $R --chain-per-warp --chain-block $b --chain-producer-grid 296 > gpurun_out/m17/n2_w_b${b}_pg296.json 2> gpurun_out/m17/n2_w_b${b}_pg296.err
done
for f in gpurun_out/m17/n2_*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'], d['roofline_nvlink'].get('same_run_nccl_allgather_busbw'))"; done
