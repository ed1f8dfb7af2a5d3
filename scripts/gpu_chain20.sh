mkdir -p gpurun_out/m20
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m20/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "chain_oneshot" > gpurun_out/m20/pytest_multi.log 2>&1; echo "pytest multi $?"; tail -1 gpurun_out/m20/pytest_multi.log
R="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --mode chain"
for b in 8192 12288; do $R --chain-oneshot --chain-block $b > gpurun_out/m20/os_b${b}.json 2>/dev/null; done
for f in gpurun_out/m20/*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'])"; done
