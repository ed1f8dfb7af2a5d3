# multi-GPU session: parity of the NCCL and P2P exchanges, then M3 benches at every available N
set -x
NG=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1; echo "pytest multi $?"; tail -15 gpurun_out/pytest_multi.log
for n in 2 4 8; do
  if [ $n -le $NG ]; then
    for m in p2p nccl allreduce; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 20 --warmup 5 --mode $m $([ $m = allreduce ] && echo --no-e2e) > gpurun_out/bench_n${n}_$m.json 2> gpurun_out/bench_n${n}_$m.err; echo "bench n=$n $m $?"; tail -c 2500 gpurun_out/bench_n${n}_$m.json; tail -3 gpurun_out/bench_n${n}_$m.err
    done
  fi
done
