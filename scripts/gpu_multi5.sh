set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "chain or range or flags" > gpurun_out/pytest_chain1.log 2>&1; echo "pytest chain1 $?"; tail -3 gpurun_out/pytest_chain1.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "chain" > gpurun_out/pytest_multi.log 2>&1; echo "pytest multi $?"; tail -3 gpurun_out/pytest_multi.log
for n in 2 4; do
  R="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 20 --warmup 5 --no-e2e --mode chain"
  for k in 8 16 32 64; do $R --pieces $k > gpurun_out/m5_n${n}_chainf$k.json 2> gpurun_out/m5_n${n}_chainf$k.err; echo "n=$n chain flags $k $?"; done
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/m5_n2_auto.json 2> gpurun_out/m5_n2_auto.err; echo "n=2 auto $?"
