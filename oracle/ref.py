"""Second, independent oracle in numpy float32 -- TEST INFRASTRUCTURE ONLY.

Re-derives the chunk plan and one round of tall aggregation +
Nesterov from the paper's description with numpy
float32 array operations (each op is one IEEE fp32 rounding; numpy never
contracts a*b+c).  It exists only to cross-check the C oracle bit for bit on
small inputs; the GPU is compared against the C oracle.
"""
from __future__ import annotations

import numpy as np


def chunk_plan(key_sizes, chunk_bytes=32768):
    ce = chunk_bytes // 4
    rows = []
    for k, nk in enumerate(key_sizes):
        off = 0
        while off < nk:
            rows.append((len(rows), k, off, min(ce, nk - off)))
            off += ce
    a = np.array(rows, dtype=np.uint64).reshape(-1, 4)
    return dict(vkey_id=a[:, 0].astype(np.uint32), key_id=a[:, 1].astype(np.uint32),
                offset=a[:, 2], length=a[:, 3])


def round_(key_sizes, grads, w, v, lr, mu, rescale=0.0, chunk_bytes=32768):
    f32 = np.float32
    N = len(grads)
    resc = f32(1.0) / f32(N) if rescale == 0.0 else f32(rescale)
    lr, mu = f32(lr), f32(mu)
    plan = chunk_plan(key_sizes, chunk_bytes)
    starts = np.concatenate([[0], np.cumsum(np.asarray(key_sizes, dtype=np.int64))])
    w2 = np.array(w, dtype=f32, copy=True)
    v2 = np.array(v, dtype=f32, copy=True)
    agg = np.zeros_like(w2)
    for k, off, ln in zip(plan["key_id"], plan["offset"], plan["length"]):
        a = int(starts[int(k)] + int(off))
        b = a + int(ln)
        merge = np.zeros(b - a, f32)                 # zeroed merge buffer
        for g in grads:                              # worker-id order (reading R3)
            merge = (merge + g[a:b]).astype(f32)
        gg = (merge * resc).astype(f32)
        vn = ((mu * v2[a:b]).astype(f32) + gg).astype(f32)
        t3 = (gg + (mu * vn).astype(f32)).astype(f32)
        w2[a:b] = (w2[a:b] - (lr * t3).astype(f32)).astype(f32)
        v2[a:b] = vn
        agg[a:b] = merge
    return w2, v2, agg


def hier_round(key_sizes, rack_grads, w, v, lr, mu, rescale=0.0):
    """Hierarchical reduction (reading R17), whole-array
    numpy float32: per rack the worker-order sum from +0, then the racks'
    sums added one rack after another from +0, then the same optimizer."""
    f32 = np.float32
    R, P = len(rack_grads), len(rack_grads[0])
    resc = f32(1.0) / f32(R * P) if rescale == 0.0 else f32(rescale)
    lr, mu = f32(lr), f32(mu)
    total = np.zeros(int(sum(key_sizes)), f32)
    for rack in rack_grads:                          # step 2: rack by rack, in rack order
        s_r = np.zeros_like(total)                   # step 1: this rack's own merge buffer
        for g in rack:
            s_r = (s_r + g).astype(f32)
        total = (total + s_r).astype(f32)
    gg = (total * resc).astype(f32)                  # step 3: the optimizer
    vn = ((mu * np.asarray(v, f32)).astype(f32) + gg).astype(f32)
    t3 = (gg + (mu * vn).astype(f32)).astype(f32)
    wn = (np.asarray(w, f32) - (lr * t3).astype(f32)).astype(f32)
    return wn, vn, total
