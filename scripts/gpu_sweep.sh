# single-GPU session: ablations + sweeps (VGG-19 / ResNet-269) and ncu of the small kernels
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
B="timeout 300 python bench.py --no-e2e --no-cpu --warmup 5"
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "replica or shared or bulk or variants" > gpurun_out/pytest_replica.log 2>&1; echo "pytest replica $?"; tail -3 gpurun_out/pytest_replica.log
for g in 148 296 592 1184 2368; do $B --steps 30 --grid $g > gpurun_out/sw_grid_$g.json 2>&1; echo "grid $g $?"; done
$B --steps 30 --kernel bulk > gpurun_out/sw_bulk_vgg.json 2>&1; echo "bulk vgg $?"
for c in enabled bypass; do $B --steps 30 --cache $c > gpurun_out/sw_cache_$c.json 2>&1; echo "cache $c $?"; done
for cb in 4096 8192 16384 32768 65536 131072 262144 524288 1048576; do
  $B --steps 30 --config resnet269 --chunk-bytes $cb > gpurun_out/sw_chunk_auto_$cb.json 2>&1; echo "chunk auto $cb $?"
  $B --steps 30 --config resnet269 --chunk-bytes $cb --kernel tiles > gpurun_out/sw_chunk_tiles_$cb.json 2>&1; echo "chunk tiles $cb $?"
done
for k in auto flat128 tiles wide bulk; do $B --steps 30 --kernel $k --config resnet50 > gpurun_out/sw_kern_rn50_$k.json 2>&1; echo "rn50 $k $?"; done
$B --steps 200 --config tiny --graph > gpurun_out/sw_tiny_graph.json 2>&1; echo "tiny graph $?"
# ncu: tiny kernel and the chunk-tile kernel at 4 KB chunks (each plain run first)
$B --steps 3 --config tiny > gpurun_out/plain_tiny.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_flat -s 3 -c 1 -o gpurun_out/prof_tiny python bench.py --no-e2e --no-cpu --warmup 5 --steps 3 --config tiny > gpurun_out/ncu_tiny.log 2>&1; echo "ncu tiny $?"
$B --steps 3 --config resnet269 --chunk-bytes 4096 --kernel tiles > gpurun_out/plain_tiles.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_tiles -s 3 -c 1 -o gpurun_out/prof_tiles4k python bench.py --no-e2e --no-cpu --warmup 5 --steps 3 --config resnet269 --chunk-bytes 4096 --kernel tiles > gpurun_out/ncu_tiles.log 2>&1; echo "ncu tiles $?"
