set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python scripts/sanitize_target.py > gpurun_out/san_plain.log 2>&1; echo "plain $?"; cat gpurun_out/san_plain.log
timeout 300 build/phub_c_example > gpurun_out/c_example.log 2>&1; echo "c example $?"; cat gpurun_out/c_example.log
timeout 600 python scripts/sanitize_target.py > gpurun_out/san_plain2.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 3 python scripts/sanitize_target.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck $?"; tail -20 gpurun_out/san_memcheck.log
