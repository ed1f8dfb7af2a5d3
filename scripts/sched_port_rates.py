"""Per-rank NVLink port rates over the round from a scripts/sched_trace.py
trace (bytes of each item spread over its work interval, 100-us bins; G from
the trace files, W = 8 / G).  usage: python scripts/sched_port_rates.py TRACE_DIR"""
import numpy as np, sys
import glob
d0 = sys.argv[1]
G = len(glob.glob(f'{d0}/trace_rank*.npz'))
W = 8 // G
data=[np.load(f'{d0}/trace_rank{r}.npz') for r in range(G)]
BIN=100
nb=22
out=np.zeros((G,G,nb)); 
for r,d in enumerate(data):
    t=d['t'].astype(np.int64); t0=t[:,0].min()
    ty=d['type']; dst=d['dst']; n=(d['hi']-d['lo'])
    bounds=d['bounds']
    for i in range(len(ty)):
        s=(t[i,1]-t0)/1e3; e=(t[i,2]-t0)/1e3
        if ty[i]==1: byt=W*4*n[i]; dd=[dst[i]]
        elif ty[i]==2 and dst[i]>=0: byt=4*n[i]; dd=[dst[i]]
        else:
            byt=4*n[i]; dd=[q for q in range(G) if q!=r]  # replicas
        for q in dd:
            # spread uniformly over [s,e]
            b0=int(s//BIN); b1=int(e//BIN)
            span=max(e-s,1e-3)
            for b in range(b0,min(b1+1,nb)):
                lo=max(s,b*BIN); hi=min(e,(b+1)*BIN)
                if hi>lo: out[r,q,b]+=byt*(hi-lo)/span
rate=out/(BIN*1e-6)/1e9  # GB/s
for r in range(G):
    print('rank',r,'OUT GB/s per bin', np.round(rate[r].sum(0)).astype(int).tolist())
for q in range(G):
    print('rank',q,'IN  GB/s per bin', np.round(rate[:,q].sum(0)).astype(int).tolist())
