# chain G = 2: one-shot consumer (one CTA per 2048 elements, hardware-ordered).
mkdir -p gpurun_out/m19
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m19/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "block_streaming" > gpurun_out/m19/pytest_1gpu.log 2>&1; echo "pytest 1gpu $?"; tail -1 gpurun_out/m19/pytest_1gpu.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "chain_oneshot or (chain and bit_exact and not pull and not flags and not barrier and not warp and not window)" > gpurun_out/m19/pytest_multi.log 2>&1; echo "pytest multi $?"; tail -1 gpurun_out/m19/pytest_multi.log
R="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --mode chain"
for rep in 1 2; do
$R > gpurun_out/m19/base_r$rep.json 2>/dev/null
for b in 8192 12288 16384 32768; do $R --chain-oneshot --chain-block $b > gpurun_out/m19/os_b${b}_r$rep.json 2>/dev/null; done
done
for f in gpurun_out/m19/*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'])"; done
