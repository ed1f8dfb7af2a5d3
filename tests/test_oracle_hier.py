"""Pins for the oracle's hierarchical-reduction round (-m "not gpu"; SURVEY
8(f) NEXT-4; reading R17).

  * two-level grouping ...... a hand-computed case where the rack-grouped sum
    differs from the flat worker-order sum (1 + 2^-23 vs 1);
  * reductions to the flat oracle ... one rack (R = 1) and one worker per rack
    (P = 1) are bit-identical to oracle.round_;
  * exactness ................ dyadic inputs sum exactly in any grouping and
    equal the float64 sum;
  * per-element form ......... hier_elems == hier_round at every element.
"""
import numpy as np
import pytest

import oracle
from workloads import manifest, values_np, dyadic_np, grad_stream

f32 = np.float32


def bits(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


def _racks(sizes, R, P, seed=0):
    E = int(sum(sizes))
    racks = [[values_np(grad_stream(r * P + k) + 37 * seed, 0, E, 25) for k in range(P)]
             for r in range(R)]
    return racks, values_np(1 + 37 * seed, 0, E, 20), values_np(2 + 37 * seed, 0, E, 25)


def test_grouping_differs_from_flat_order():
    """rack 0 = [1, 0], rack 1 = [2^-24, 2^-24]: flat ((((0+1)+0)+2^-24)+2^-24) = 1
    (each 1 + 2^-24 ties to even); grouped: S_0 = 1, S_1 = 2^-23, s = 1 + 2^-23."""
    t = f32(2.0 ** -24)
    racks = [[np.array([1], f32), np.array([0], f32)], [np.array([t], f32), np.array([t], f32)]]
    z = np.zeros(1, f32)
    _, _, s = oracle.hier_round([1], racks, z, z, 0.0, 0.0)
    assert bits(s)[0] == 0x3F800001                       # 1 + 2^-23
    _, _, sf = oracle.round_([1], [g for r in racks for g in r], z, z, 0.0, 0.0)
    assert bits(sf)[0] == 0x3F800000                      # flat worker order: 1
    # the optimizer sees s * 1/(R*P): v' = s/4 with mu = 0, w' = -lr * v'
    w, v, _ = oracle.hier_round([1], racks, z, z, 1.0, 0.0)
    assert v[0] == f32(f32(1 + 2.0 ** -23) * f32(0.25)) and w[0] == -v[0]


@pytest.mark.parametrize("name,P", [("tiny", 4), ("small", 3)])
def test_one_rack_is_the_flat_round(name, P):
    sizes = manifest(name) if name != "small" else [3, 3, 9408, 64, 7]
    racks, w0, v0 = _racks(sizes, 1, P, seed=3)
    hw, hv, hs = oracle.hier_round(sizes, racks, w0, v0, 0.1, 0.9)
    fw, fv, fs = oracle.round_(sizes, racks[0], w0, v0, 0.1, 0.9)
    for a, b in ((hw, fw), (hv, fv), (hs, fs)):
        assert np.array_equal(bits(a), bits(b))


def test_one_worker_per_rack_is_the_flat_round():
    sizes = [1000, 8192, 3, 40000]
    racks, w0, v0 = _racks(sizes, 5, 1, seed=4)
    racks[2][0][:50] = -0.0                               # signed zeros survive the +0 starts
    hw, hv, hs = oracle.hier_round(sizes, racks, w0, v0, 0.1, 0.9, chunk_bytes=4096)
    fw, fv, fs = oracle.round_(sizes, [r[0] for r in racks], w0, v0, 0.1, 0.9, chunk_bytes=4096)
    for a, b in ((hw, fw), (hv, fv), (hs, fs)):
        assert np.array_equal(bits(a), bits(b))


def test_dyadic_inputs_equal_exact_sum():
    sizes = [5000, 123, 70000]
    E = sum(sizes)
    R, P = 3, 4
    racks = [[dyadic_np(100 + r * P + k, E) for k in range(P)] for r in range(R)]
    exact = np.sum([g.astype(np.float64) for rack in racks for g in rack], axis=0)
    z = np.zeros(E, f32)
    _, _, s = oracle.hier_round(sizes, racks, z, z, 0.1, 0.9)
    assert np.array_equal(s.astype(np.float64), exact)


def test_hier_elems_matches_round():
    sizes = manifest("tiny")
    racks, w0, v0 = _racks(sizes, 4, 2, seed=5)
    w, v, s = oracle.hier_round(sizes, racks, w0, v0, 0.1, 0.9)
    idx = np.array([0, 1, 1023, 1024, 9000, 288767])
    g = np.stack([np.stack([racks[r][k][idx] for k in range(2)]) for r in range(4)])
    ew, ev, es = oracle.hier_elems(g, w0[idx], v0[idx], 0.1, 0.9)
    for a, b in ((ew, w[idx]), (ev, v[idx]), (es, s[idx])):
        assert np.array_equal(bits(a), bits(b))


@pytest.mark.parametrize("R,P", [(2, 4), (3, 2), (4, 1), (1, 5)])
def test_independent_numpy_oracle_agrees(R, P):
    """oracle/ref.py re-derives the hierarchical round with whole-array numpy
    fp32 ops (no chunking, no C); it must agree with the C oracle bit for bit."""
    from oracle import ref
    sizes = [1000, 33, 70000, 3]
    racks, w0, v0 = _racks(sizes, R, P, seed=6 + R)
    cw, cv, cs = oracle.hier_round(sizes, racks, w0, v0, 0.1, 0.9, chunk_bytes=4096)
    nw, nv, ns = ref.hier_round(sizes, racks, w0, v0, 0.1, 0.9)
    for a, b in ((cw, nw), (cv, nv), (cs, ns)):
        assert np.array_equal(bits(a), bits(b))
