set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1; echo "pytest multi $?"; tail -3 gpurun_out/pytest_multi.log
for n in 2 4; do
  R="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 30 --warmup 5"
  $R > gpurun_out/m6_n${n}_auto.json 2> gpurun_out/m6_n${n}_auto.err; echo "n=$n auto $?"
done
