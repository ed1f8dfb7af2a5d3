set -x
NG=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1; echo "pytest multi $?"; tail -3 gpurun_out/pytest_multi.log
for n in 2 4; do
    R="timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 20 --warmup 5 --no-e2e --mode p2p"
    $R > gpurun_out/m3_n${n}_default.json 2> gpurun_out/m3_n${n}_default.err; echo "n=$n default $?"
    for mb in 1 2; do $R --minb $mb > gpurun_out/m3_n${n}_minb$mb.json 2>&1; echo "n=$n minb $mb $?"; done
    for g in 296 1184 2368; do $R --grid $g > gpurun_out/m3_n${n}_grid$g.json 2>&1; echo "n=$n grid $g $?"; done
    $R --seg 256 > gpurun_out/m3_n${n}_seg256.json 2>&1; echo "n=$n seg $?"
    $R --kernel bulk > gpurun_out/m3_n${n}_bulk.json 2>&1; echo "n=$n bulk $?"
done
