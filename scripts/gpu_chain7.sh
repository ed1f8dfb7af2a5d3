# Round 1, session 2: block-streaming chain (one launch per rank, per-block flags).
set -x
mkdir -p gpurun_out/m7
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m7/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "block_streaming or stage_flags or chain" > gpurun_out/m7/pytest_1gpu.log 2>&1; echo "pytest 1gpu $?"; tail -3 gpurun_out/m7/pytest_1gpu.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "chain" > gpurun_out/m7/pytest_multi.log 2>&1; echo "pytest multi $?"; tail -3 gpurun_out/m7/pytest_multi.log
R="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --mode chain"
$R > gpurun_out/m7/n2_blocks32k.json 2> gpurun_out/m7/n2_blocks32k.err; echo "blocks32k $?"
$R --chain-block 16384 > gpurun_out/m7/n2_blocks16k.json 2> gpurun_out/m7/n2_blocks16k.err; echo "blocks16k $?"
$R --chain-block 65536 > gpurun_out/m7/n2_blocks64k.json 2> gpurun_out/m7/n2_blocks64k.err; echo "blocks64k $?"
$R --chain-block 8192 > gpurun_out/m7/n2_blocks8k.json 2> gpurun_out/m7/n2_blocks8k.err; echo "blocks8k $?"
$R --chain-pull > gpurun_out/m7/n2_blocks32k_pull.json 2> gpurun_out/m7/n2_blocks32k_pull.err; echo "pull $?"
$R --chain-sync flags > gpurun_out/m7/n2_flags8.json 2> gpurun_out/m7/n2_flags8.err; echo "flags $?"
grep -h '"value"' gpurun_out/m7/n2_*.json | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'], d['config']['mode'][-80:])"
