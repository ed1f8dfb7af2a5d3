# e2e copy streams per direction at N = 1.
mkdir -p gpurun_out/m16
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m16/build.log 2>&1
for k in 1 2 4; do
  timeout 600 python bench.py --no-cpu --steps 10 --e2e-steps 4 --e2e-streams $k > gpurun_out/m16/e2e_s$k.json 2> gpurun_out/m16/e2e_s$k.err
done
for f in gpurun_out/m16/e2e_*.json; do echo -n "$f "; grep -h '"value"' $f | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['e2e'])"; done
