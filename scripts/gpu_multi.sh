# multi-GPU session: parity of the NCCL exchange, then M3 benches at every available N
set -x
nvidia-smi --query-gpu=index,name --format=csv
NG=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1; echo "pytest multi $?"; tail -15 gpurun_out/pytest_multi.log
for n in 2 4 8; do
  if [ $n -le $NG ]; then
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err; echo "bench n=$n $?"; tail -c 2500 gpurun_out/bench_n$n.json; tail -3 gpurun_out/bench_n$n.err
  fi
done
