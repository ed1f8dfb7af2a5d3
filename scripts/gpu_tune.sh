# single-GPU tuning session: flat-kernel schedules / occupancy builds, tile sizes, bulk
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/pytest_gpu.log
B="timeout 300 python bench.py --no-e2e --no-cpu --warmup 5 --steps 40"
for cfg in vgg19 resnet269; do
 for rep in 1 2; do
  $B --config $cfg > gpurun_out/tu_${cfg}_default_$rep.json 2>&1
  for seg in 64 256 1024; do $B --config $cfg --seg $seg > gpurun_out/tu_${cfg}_seg${seg}_$rep.json 2>&1; done
  for mb in 1 2 4 6; do $B --config $cfg --minb $mb > gpurun_out/tu_${cfg}_minb${mb}_$rep.json 2>&1; $B --config $cfg --minb $mb --seg 256 > gpurun_out/tu_${cfg}_minb${mb}_seg256_$rep.json 2>&1; done
  for te in 1024 2048 4096 8192; do $B --config $cfg --kernel tiles --tile-elems $te > gpurun_out/tu_${cfg}_tiles${te}_$rep.json 2>&1; done
  $B --config $cfg --kernel bulk > gpurun_out/tu_${cfg}_bulk_$rep.json 2>&1
 done
done
echo done
