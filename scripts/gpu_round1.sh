set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench exit $?"; tail -c 3000 gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
for k in flat flat128 tiles wide; do timeout 300 python bench.py --steps 30 --warmup 5 --kernel $k --no-e2e --no-cpu > gpurun_out/bench_$k.json 2>&1; echo "$k $?"; done
for c in resnet50 alexnet resnet269 tiny; do timeout 300 python bench.py --steps 30 --warmup 5 --config $c --no-e2e --no-cpu > gpurun_out/bench_cfg_$c.json 2>&1; echo "$c $?"; done
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 $?"
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_flat -s 3 -c 1 -o gpurun_out/prof_flat python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "ncu2 $?"
ls -la gpurun_out
