# single-GPU evidence session: full GPU tests, smoke, default bench, reference arm, ncu of the default kernel
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/f_pytest_gpu.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/f_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke $?"
timeout 600 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench $?"; tail -c 1500 gpurun_out/f_bench.json
timeout 600 python bench.py --impl reference > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err; echo "ref $?"; tail -c 800 gpurun_out/f_bench_ref.json
timeout 300 python bench.py --config tiny --graph --steps 200 --no-e2e --no-cpu > gpurun_out/f_tiny.json 2>&1; echo "tiny $?"
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/f_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/f_ncu1.log 2>&1; echo "ncu launches $?"
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/f_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_flat -s 3 -c 1 -o gpurun_out/f_prof_flat python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/f_ncu2.log 2>&1; echo "ncu full $?"
