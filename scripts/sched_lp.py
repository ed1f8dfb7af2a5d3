"""Byte-balancing model of the scheduled exchange: choose, per
owner o, the share of the model it owns and how much of that share is
exchanged RAW (every other rank stores its W raw worker slices into o) or as a
CHAIN (the worker-order partial travels rank 0 -> 1 -> ... -> G-1, and the
last rank stores the finished sum into o unless o is the last rank), so that
the busiest NVLink port -- max over GPUs and directions of the bytes it moves,
replica stores of w' included -- is minimal.  Units: model sizes (4E bytes).

    python scripts/sched_lp.py        # prints SCHED_TABLE for sharded.py

Only this offline script needs scipy; sharded.py carries the table and a
plain-Python byte count of any (weights, raw fractions) it is given.
"""
import numpy as np
from scipy.optimize import linprog


def port_rows(G, W):
    """Linear port loads in the variables x[o, s] (s = 0 RAW, 1 CHAIN)."""
    nv = 2 * G
    L = {(g, d): np.zeros(nv) for g in range(G) for d in ("in", "out")}
    for o in range(G):
        raw, ch = 2 * o, 2 * o + 1
        for q in range(G):
            if q != o:
                L[(o, "in")][raw] += W          # W raw slices from every other rank
                L[(q, "out")][raw] += W
        for p in range(G - 1):                  # the partial's hops
            L[(p, "out")][ch] += 1
            L[(p + 1, "in")][ch] += 1
        if o != G - 1:                          # the finished sum to the owner
            L[(G - 1, "out")][ch] += 1
            L[(o, "in")][ch] += 1
        for v in (raw, ch):                     # w' into every other replica
            for q in range(G):
                if q != o:
                    L[(o, "out")][v] += 1
                    L[(q, "in")][v] += 1
    return L


def solve(G, W):
    L = port_rows(G, W)
    nv = 2 * G + 1
    A = [np.r_[row, -1.0] for row in L.values()]
    res = linprog(np.r_[np.zeros(2 * G), 1.0], A_ub=A, b_ub=np.zeros(len(A)),
                  A_eq=[np.r_[np.ones(2 * G), 0.0]], b_eq=[1.0], bounds=[(0, None)] * nv)
    x = res.x[:-1]
    wts = [x[2 * o] + x[2 * o + 1] for o in range(G)]
    rf = [x[2 * o] / wts[o] if wts[o] > 1e-9 else 0.0 for o in range(G)]
    return res.x[-1], wts, rf


if __name__ == "__main__":
    print("SCHED_TABLE = {")
    for G in (2, 3, 4, 8):
        W = 8 // G if 8 % G == 0 else 3
        t, wts, rf = solve(G, W)
        push = 1 + (G * W - W - 1) / G
        print(f"    {G}: ({[round(float(w), 4) + 0.0 for w in wts]}, {[round(float(r), 4) + 0.0 for r in rf]}),"
              f"  # W={W}: busiest port {t:.4f} vs push exchange {push:.4f} model sizes")
    print("}")
