# Start barriers restored: push / hierarchical parity at G = 2 and 4.
mkdir -p gpurun_out/m29
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m29/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider -k "bit_exact and (push or hier)" > gpurun_out/m29/pytest_multi.log 2>&1; echo "pytest multi $?"; tail -1 gpurun_out/m29/pytest_multi.log
