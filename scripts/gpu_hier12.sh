# Round 1, session 2: hierarchical exchange with one rack (G = 1) + ncu of k_hier.
set -x
mkdir -p gpurun_out/m12
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m12/build.log 2>&1
timeout 300 python bench.py --mode hier --no-e2e --steps 30 > gpurun_out/m12/n1_hier.json 2> gpurun_out/m12/n1_hier.err; echo "hier1 $?"
timeout 300 python bench.py --no-e2e --no-cpu --steps 30 > gpurun_out/m12/n1_default.json 2> gpurun_out/m12/n1_default.err; echo "default $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_hier -s 5 -c 1 -o gpurun_out/m12/prof_k_hier python bench.py --mode hier --no-e2e --steps 3 --warmup 5 > gpurun_out/m12/ncu_hier.log 2>&1; echo "ncu $?"
cat gpurun_out/m12/n1_hier.json gpurun_out/m12/n1_default.json | grep value | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['ms_per_step'])"
