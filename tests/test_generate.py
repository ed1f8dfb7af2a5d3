"""Pins for the input generator's full-mantissa recipe (-m "not gpu").

The GPU parity tests draw gradients, weights and momenta from
workloads.generate.fullmant_*: a random 24-bit significand, a random binade
2^-e (e in [0, 30]) and a random sign per element.  These tests fix the two
properties the parity argument rests on:

* numpy (oracle side) and torch (device side) produce identical bits;
* the inputs DISCRIMINATE summation order -- a kernel that summed the workers
  in any order other than worker-id order (reversed, pairwise tree, rotated)
  would differ from the worker-order oracle on most elements (SPEC.md:224,
  DESIGN.md reading R3), which the legacy 17-bit recipe could not show
  (its sums are exact in any order).
"""
import numpy as np
import pytest

from workloads import grad_stream, values_np
from workloads.generate import fullmant_at_np, fullmant_np

f32 = np.float32
torch = pytest.importorskip("torch")


def bits(a):
    return np.asarray(a, dtype=f32).view(np.uint32)


def test_numpy_and_torch_agree_bit_for_bit():
    from workloads.generate import fullmant_torch
    for stream, start, n in ((1000, 0, 100003), (1007, 123456789, 5000), (2, 1 << 40, 4096)):
        a = fullmant_np(stream, start, n)
        b = fullmant_torch(stream, start, n, "cpu", block=1 << 14).numpy()
        assert np.array_equal(bits(a), bits(b))
    idx = np.array([0, 5, 99999, 1 << 33], np.uint64)
    assert np.array_equal(bits(fullmant_at_np(1003, idx)),
                          bits(np.array([fullmant_np(1003, int(i), 1)[0] for i in idx], f32)))


def test_values_are_normal_full_mantissa_both_signs():
    a = fullmant_np(1001, 0, 1 << 18)
    mag = np.abs(a.astype(np.float64))
    assert np.all(np.isfinite(a)) and mag.min() >= 2.0 ** -30 and mag.max() < 2.0
    assert 0.45 < np.mean(a < 0) < 0.55
    e = (bits(a) >> 23) & 0xFF
    assert set(np.unique(127 - e.astype(np.int64)).tolist()) == set(range(31))
    # the low mantissa bits are populated (a 17-bit-significand recipe leaves them 0)
    assert np.mean((bits(a) & 0x7F) != 0) > 0.95


def _sum(grads, order):
    s = np.zeros_like(grads[0])
    for k in order:
        s = (s + grads[k]).astype(f32)
    return s


def _tree(grads):
    xs = list(grads)
    while len(xs) > 1:
        xs = [(xs[i] + xs[i + 1]).astype(f32) if i + 1 < len(xs) else xs[i]
              for i in range(0, len(xs), 2)]
    return xs[0]


@pytest.mark.parametrize("N", [3, 8, 33])
def test_full_mantissa_inputs_discriminate_summation_order(N):
    E = 20000
    g = [fullmant_np(grad_stream(w), 0, E) for w in range(N)]
    ref = _sum(g, range(N))
    # (with 3 terms only the first pairing can differ: ~20 %; with 8 or more, a third to most)
    floor = 0.15 if N < 8 else 0.25
    others = [_sum(g, reversed(range(N))), _sum(g, list(range(1, N)) + [0])]
    if N > 3:                                     # a 3-leaf pairwise tree IS worker order
        others.append(_tree(g))
    for other in others:
        assert np.mean(bits(other) != bits(ref)) > floor


@pytest.mark.parametrize("N", [3, 8, 33])
def test_legacy_recipe_is_order_blind(N):
    """Why the legacy 17-bit recipe is kept only for bandwidth runs: its sums are
    exact, so every order gives the float64 sum."""
    E = 20000
    g = [values_np(grad_stream(w), 0, E, 25) for w in range(N)]
    exact = np.sum(np.stack(g).astype(np.float64), axis=0)
    for s in (_sum(g, range(N)), _sum(g, reversed(range(N))), _tree(g)):
        assert np.array_equal(s.astype(np.float64), exact)
