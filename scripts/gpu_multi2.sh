set -x
NG=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1; echo "pytest multi $?"; tail -3 gpurun_out/pytest_multi.log
for n in 2 4; do
  if [ $n -le $NG ]; then
    R="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 20 --warmup 5"
    $R --mode p2p > gpurun_out/m2_n${n}_p2p.json 2> gpurun_out/m2_n${n}_p2p.err; echo "n=$n p2p $?"
    $R --mode p2p --oneshot 0 --no-e2e > gpurun_out/m2_n${n}_p2p_persist.json 2> gpurun_out/m2_n${n}_p2p_persist.err; echo "n=$n p2p persist $?"
    $R --mode p2p --kernel flat128 --no-e2e > gpurun_out/m2_n${n}_p2p_v4.json 2> gpurun_out/m2_n${n}_p2p_v4.err; echo "n=$n p2p v4 $?"
    $R --mode nccl --no-e2e > gpurun_out/m2_n${n}_nccl.json 2> gpurun_out/m2_n${n}_nccl.err; echo "n=$n nccl $?"
  fi
done
