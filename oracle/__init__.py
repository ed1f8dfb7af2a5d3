"""CPU oracle for the PHub hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_1805_07891_b200``) never imports it and shares no code with it.

Two independent implementations live here:

* ``phub_oracle.c`` (ctypes, this module): plain C scalar loops, built with
  ``-ffp-contract=off`` -- the oracle the GPU is compared against;
* ``ref.py``: a numpy float32 re-derivation used only to cross-check the C
  oracle bit for bit on small inputs.

See the header of ``phub_oracle.c`` for each function's paper citation and the
pins in ``tests/test_oracle_*.py``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "phub_oracle.c")
_LIB = os.path.join(_HERE, "libphub_oracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
          "-shared", "-fPIC"]


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = C.CDLL(build())
            u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")
            u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
            i32p = np.ctypeslib.ndpointer(np.int32, flags="C")
            f32p = np.ctypeslib.ndpointer(np.float32, flags="C")
            lib.oracle_chunk_count.argtypes = [u64p, C.c_int32, C.c_uint64]
            lib.oracle_chunk_count.restype = C.c_int64
            lib.oracle_chunk_plan.argtypes = [u64p, C.c_int32, C.c_uint64, u32p, u32p, u64p,
                                              u64p, C.c_uint64]
            lib.oracle_chunk_plan.restype = C.c_int64
            lib.oracle_owners_lpt.argtypes = [u64p, C.c_uint64, C.c_int32, i32p]
            lib.oracle_owners_contig.argtypes = [u64p, C.c_uint64, C.c_int32, i32p]
            lib.oracle_bruteforce_max_load.argtypes = [u64p, C.c_uint64, C.c_int32]
            lib.oracle_bruteforce_max_load.restype = C.c_int64
            lib.oracle_round.argtypes = [u64p, C.c_int32, C.c_uint64, C.c_int32,
                                         C.POINTER(C.c_void_p), f32p, f32p, C.c_void_p,
                                         C.c_float, C.c_float, C.c_float, C.c_void_p,
                                         C.c_int32]
            lib.oracle_elems.argtypes = [C.c_uint64, C.c_int32, f32p, f32p, f32p, C.c_void_p,
                                         C.c_float, C.c_float, C.c_float]
            lib.oracle_elems.restype = None
            lib.oracle_hier_round.argtypes = [u64p, C.c_int32, C.c_uint64, C.c_int32, C.c_int32,
                                              C.POINTER(C.c_void_p), f32p, f32p, C.c_void_p,
                                              C.c_float, C.c_float, C.c_float]
            lib.oracle_hier_elems.argtypes = [C.c_uint64, C.c_int32, C.c_int32, f32p, f32p, f32p,
                                              C.c_void_p, C.c_float, C.c_float, C.c_float]
            lib.oracle_hier_elems.restype = None
            lib.oracle_max_threads.restype = C.c_int
            _lib = lib
    return _lib


class OracleError(RuntimeError):
    pass


def _u64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def chunk_count(key_sizes, chunk_bytes: int = 32768) -> int:
    r = _load().oracle_chunk_count(_u64(key_sizes), len(key_sizes), chunk_bytes)
    if r < 0:
        raise OracleError(f"oracle_chunk_count -> {r}")
    return int(r)


def chunk_plan(key_sizes, chunk_bytes: int = 32768) -> dict:
    """vkey table: dict of arrays vkey_id, key_id, offset, length."""
    n = _u64(key_sizes)
    cnt = chunk_count(n, chunk_bytes)
    out = dict(vkey_id=np.zeros(cnt, np.uint32), key_id=np.zeros(cnt, np.uint32),
               offset=np.zeros(cnt, np.uint64), length=np.zeros(cnt, np.uint64))
    r = _load().oracle_chunk_plan(n, len(n), chunk_bytes, out["vkey_id"], out["key_id"],
                                  out["offset"], out["length"], cnt)
    if r != cnt:
        raise OracleError(f"oracle_chunk_plan -> {r}")
    return out


def owners_lpt(lengths, G: int) -> np.ndarray:
    L = _u64(lengths)
    o = np.full(len(L), -1, np.int32)
    if _load().oracle_owners_lpt(L, len(L), G, o) != 0:
        raise OracleError("oracle_owners_lpt")
    return o


def owners_contig(lengths, G: int) -> np.ndarray:
    L = _u64(lengths)
    o = np.full(len(L), -1, np.int32)
    if _load().oracle_owners_contig(L, len(L), G, o) != 0:
        raise OracleError("oracle_owners_contig")
    return o


def bruteforce_max_load(lengths, G: int) -> int:
    L = _u64(lengths)
    r = _load().oracle_bruteforce_max_load(L, len(L), G)
    if r < 0:
        raise OracleError("instance too large for brute force (S:100)")
    return int(r)


def canonical_text(plan: dict, owners) -> str:
    """S:125 canonical text, one owner column: vkey_id,key_id,offset,length,owner."""
    rows = zip(plan["vkey_id"].tolist(), plan["key_id"].tolist(), plan["offset"].tolist(),
               plan["length"].tolist(), np.asarray(owners).tolist())
    return "".join(f"{a},{b},{c},{d},{e}\n" for a, b, c, d, e in rows)


def round_(key_sizes, grads, w, v, lr: float, mu: float, rescale: float = 0.0,
           chunk_bytes: int = 32768, keep_agg: bool = True, order=None, nthreads: int = 1):
    """One push/aggregate/optimize round.

    grads: sequence of N float32 arrays of E elements (key-major, unpadded).
    Returns (w', v', s) as new arrays (inputs are not modified); s is None
    unless keep_agg.
    """
    n = _u64(key_sizes)
    E = int(n.sum())
    gs = [np.ascontiguousarray(g, dtype=np.float32) for g in grads]
    for g in gs:
        if g.shape != (E,):
            raise OracleError("gradient length != E")
    N = len(gs)
    ptrs = (C.c_void_p * N)(*[g.ctypes.data for g in gs])
    w2 = np.array(w, dtype=np.float32, copy=True)
    v2 = np.array(v, dtype=np.float32, copy=True)
    agg = np.zeros(E, np.float32) if keep_agg else None
    ordr = None
    if order is not None:
        ordr = np.ascontiguousarray(order, dtype=np.uint32)
    r = _load().oracle_round(n, len(n), chunk_bytes, N, ptrs, w2, v2,
                             agg.ctypes.data if agg is not None else None,
                             lr, mu, rescale,
                             ordr.ctypes.data if ordr is not None else None, nthreads)
    if r != 0:
        raise OracleError(f"oracle_round -> {r}")
    return w2, v2, agg


def elems(g, w, v, lr: float, mu: float, rescale: float = 0.0):
    """Per-element oracle on gathered elements: g is (N, m) worker-major."""
    g = np.ascontiguousarray(g, dtype=np.float32)
    N, m = g.shape
    w2 = np.array(w, dtype=np.float32, copy=True)
    v2 = np.array(v, dtype=np.float32, copy=True)
    s = np.zeros(m, np.float32)
    _load().oracle_elems(m, N, g.reshape(-1), w2, v2, s.ctypes.data, lr, mu, rescale)
    return w2, v2, s


def hier_round(key_sizes, rack_grads, w, v, lr: float, mu: float, rescale: float = 0.0,
               chunk_bytes: int = 32768):
    """Hierarchical reduction round (reading R17).

    rack_grads: R sequences of P float32 arrays of E elements (worker k of rack
    r).  Returns (w', v', s) with s = ((+0 + S_0) + S_1) + ... + S_{R-1} and
    S_r the worker-order sum of rack r.
    """
    n = _u64(key_sizes)
    E = int(n.sum())
    R, P = len(rack_grads), len(rack_grads[0])
    gs = [np.ascontiguousarray(g, dtype=np.float32) for rack in rack_grads for g in rack]
    if any(len(rack) != P for rack in rack_grads) or any(g.shape != (E,) for g in gs):
        raise OracleError("every rack needs P gradients of E elements")
    ptrs = (C.c_void_p * len(gs))(*[g.ctypes.data for g in gs])
    w2 = np.array(w, dtype=np.float32, copy=True)
    v2 = np.array(v, dtype=np.float32, copy=True)
    agg = np.zeros(E, np.float32)
    r = _load().oracle_hier_round(n, len(n), chunk_bytes, R, P, ptrs, w2, v2, agg.ctypes.data,
                                  lr, mu, rescale)
    if r != 0:
        raise OracleError(f"oracle_hier_round -> {r}")
    return w2, v2, agg


def hier_elems(g, w, v, lr: float, mu: float, rescale: float = 0.0):
    """hier_round's arithmetic on gathered elements: g is (R, P, m)."""
    g = np.ascontiguousarray(g, dtype=np.float32)
    R, P, m = g.shape
    w2 = np.array(w, dtype=np.float32, copy=True)
    v2 = np.array(v, dtype=np.float32, copy=True)
    s = np.zeros(m, np.float32)
    _load().oracle_hier_elems(m, R, P, g.reshape(-1), w2, v2, s.ctypes.data, lr, mu, rescale)
    return w2, v2, s


def max_threads() -> int:
    return int(_load().oracle_max_threads())
