set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/pytest_gpu.log
B="timeout 300 python bench.py --no-e2e --no-cpu --warmup 5 --steps 40"
for cfg in vgg19 resnet269 resnet50 alexnet; do
 for rep in 1 2; do
  $B --config $cfg --kernel tiles --tile-elems 1024 > gpurun_out/t2_${cfg}_tiles1024_$rep.json 2>&1
  $B --config $cfg --oneshot 1 > gpurun_out/t2_${cfg}_oneshot8_$rep.json 2>&1
  $B --config $cfg --oneshot 1 --kernel flat128 > gpurun_out/t2_${cfg}_oneshot4_$rep.json 2>&1
  $B --config $cfg > gpurun_out/t2_${cfg}_default_$rep.json 2>&1
 done
done
timeout 600 python bench.py --steps 20 --warmup 3 --e2e-steps 4 --no-cpu > gpurun_out/t2_e2e.json 2>&1; echo "e2e $?"; tail -c 600 gpurun_out/t2_e2e.json
