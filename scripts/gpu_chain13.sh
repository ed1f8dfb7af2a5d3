# Round 1, session 2: chain with producer back-pressure (L2-resident inbox + CONSUME discard).
set -x
mkdir -p gpurun_out/m13
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m13/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "chain" > gpurun_out/m13/pytest_multi.log 2>&1; echo "pytest multi $?"; tail -2 gpurun_out/m13/pytest_multi.log
R="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --mode chain"
$R > gpurun_out/m13/n2_base.json 2> gpurun_out/m13/n2_base.err
for w in 768 1024 1536 2048; do
  $R --chain-window $w > gpurun_out/m13/n2_w$w.json 2> gpurun_out/m13/n2_w$w.err
  $R --chain-window $w --chain-no-consume > gpurun_out/m13/n2_w${w}_nc.json 2> gpurun_out/m13/n2_w${w}_nc.err
done
for w in 1024 2048 3072; do
  $R --chain-block 8192 --chain-window $w > gpurun_out/m13/n2_b8k_w$w.json 2> gpurun_out/m13/n2_b8k_w$w.err
done
for f in gpurun_out/m13/n2_*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'])"; done
