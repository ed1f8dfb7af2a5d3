# ncu of the chain's block-streamed kernels on one GPU (sequential producer -> consumer).
mkdir -p gpurun_out/m25
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m25/build.log 2>&1
timeout 300 python scripts/chain_one_gpu.py > gpurun_out/m25/chain_one_gpu.txt 2>&1; echo "plain $?"; cat gpurun_out/m25/chain_one_gpu.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_blocks -s 2 -c 2 -o gpurun_out/m25/prof_k_blocks python scripts/chain_one_gpu.py --rounds 3 > gpurun_out/m25/ncu.log 2>&1; echo "ncu $?"
