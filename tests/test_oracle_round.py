"""Pins for the oracle's aggregation + Nesterov round (-m "not gpu").

What pins what (a plausible mistake in the oracle must fail one of these):
  * worker-order sum from +0.0f ... exact dyadic sums, the 1 + 2^-24 + 2^-24
    order case, the signed-zero case, S:175;
  * the NAG recurrence ............. S:193 / S:375 hex values, the multi-round
    closed form (exact for t = 1..18), mu=0 -> SGD, lr=0 identity, fixed point,
    quadratic convergence bound;
  * chunking/ordering ............... chunk-size, vkey-order and thread-count
    invariance (element-wise), the independent numpy oracle.
"""
import numpy as np
import pytest

import oracle
from oracle import ref
from workloads import manifest, values_np, dyadic_np, grad_stream
from conftest import read_golden

f32 = np.float32


def bits(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


def _inputs(sizes, N, seed=0):
    E = int(sum(sizes))
    grads = [values_np(grad_stream(w) + 37 * seed, 0, E, 25) for w in range(N)]
    w0 = values_np(1 + 37 * seed, 0, E, 20)
    v0 = values_np(2 + 37 * seed, 0, E, 25)
    return grads, w0, v0


# ------------------------------------------------------------ aggregation
def test_s175_sum():
    w, v, s = oracle.round_([2], [np.array([1, 2], f32), np.array([3, 4], f32)],
                            np.zeros(2, f32), np.zeros(2, f32), lr=0.0, mu=0.5)
    assert s.tolist() == [4.0, 6.0]
    assert v.tolist() == [2.0, 3.0]                       # mean via rescale 1/N
    assert w.tolist() == [0.0, 0.0]


def test_dyadic_sum_exact():
    # k/256 with |k| <= 1023: every partial sum is exact in fp32, so the
    # worker-order sum equals the float64 sum (SURVEY 8(c) pin table).
    sizes = [3, 700, 5000]
    E = sum(sizes)
    for N in (1, 2, 3, 5, 8, 16):
        grads = [dyadic_np(50 + w, E) for w in range(N)]
        _, _, s = oracle.round_(sizes, grads, np.zeros(E, f32), np.zeros(E, f32), 0.1, 0.9,
                                chunk_bytes=4096)
        exact = np.sum(np.stack(grads).astype(np.float64), axis=0)
        assert np.array_equal(s.astype(np.float64), exact)


def test_worker_order():
    # ((0 + 1) + 2^-24) + 2^-24 = 1 (ties to even twice); the reversed order
    # (2^-24 + 2^-24) + 1 = 1 + 2^-23.  Reading R3 fixes worker-id order.
    e = f32(2.0 ** -24)
    g = [np.array([1.0], f32), np.array([e], f32), np.array([e], f32)]
    _, _, s = oracle.round_([1], g, np.zeros(1, f32), np.zeros(1, f32), 0.0, 0.0)
    assert bits(s)[0] == bits(f32(1.0))
    _, _, s = oracle.round_([1], g[::-1], np.zeros(1, f32), np.zeros(1, f32), 0.0, 0.0)
    assert bits(s)[0] == bits(f32(1.0 + 2.0 ** -23))


def test_signed_zero_start():
    # merge buffer starts at +0.0f: +0 + (-0) = +0, so s is never -0
    for N in (1, 4):
        g = [np.array([-0.0, -0.0, 0.0], f32) for _ in range(N)]
        _, _, s = oracle.round_([3], g, np.zeros(3, f32), np.zeros(3, f32), 0.1, 0.9)
        assert bits(s).tolist() == [0, 0, 0]


def test_n1_sum_is_identity():
    g = values_np(grad_stream(0), 0, 10000, 25)
    _, _, s = oracle.round_([10000], [g], np.zeros(10000, f32), np.zeros(10000, f32), 0.1, 0.9)
    assert np.array_equal(bits(s), bits(g + f32(0.0)))


# ---------------------------------------------------------------- NAG
@pytest.mark.parametrize("row", read_golden("nag_cases.txt"), ids=lambda r: r[0])
def test_nag_golden(row):
    name, _cite, N, lr, mu, resc, w0, v0, g, ew, ev = row
    N = int(N)
    grads = [np.array([float(g)], f32) for _ in range(N)]
    if name == "s175":
        grads = [np.array([1.0], f32), np.array([3.0], f32)]
    w, v, _ = oracle.round_([1], grads, np.array([float(w0)], f32), np.array([float(v0)], f32),
                            float(lr), float(mu), float(resc))
    assert bits(w)[0] == int(ew, 16)
    assert bits(v)[0] == int(ev, 16)


def test_multi_round_closed_form():
    # g == 1 from every worker, w0 = v0 = 0, mu = lr = 1/2, rescale = 1/N:
    #   v_t = 2(1 - 2^-t),  w_t = -t + 1/2 - 2^-(t+1)   (exact in fp32 for t <= 18)
    N = 4
    w, v = np.zeros(5, f32), np.zeros(5, f32)
    ones = [np.ones(5, f32) for _ in range(N)]
    for t in range(1, 19):
        w, v, _ = oracle.round_([2, 3], ones, w, v, 0.5, 0.5)
        assert np.all(v == f32(2.0 * (1.0 - 2.0 ** -t)))
        assert np.all(w == f32(-t + 0.5 - 2.0 ** -(t + 1)))
        assert float(w[0]) == -t + 0.5 - 2.0 ** -(t + 1)      # exact, not just rounded


def test_mu0_is_sgd_and_lr0_identity():
    sizes = [1000, 33]
    grads, w0, v0 = _inputs(sizes, 1)
    w, v, s = oracle.round_(sizes, grads, w0, v0, 0.1, 0.0)
    assert np.array_equal(bits(v), bits(s))                        # v' = g (N = 1)
    assert np.array_equal(bits(w), bits(w0 - f32(0.1) * s))        # plain SGD
    for N in (1, 3, 8):
        grads, w0, v0 = _inputs(sizes, N, seed=N)
        w, _, _ = oracle.round_(sizes, grads, w0, v0, 0.0, 0.9)
        assert np.array_equal(bits(w), bits(w0))                   # lr = 0 identity (BJ)


def test_fixed_point():
    w0 = values_np(1, 0, 300, 20)
    w, v, _ = oracle.round_([300], [np.zeros(300, f32)] * 3, w0, np.zeros(300, f32), 0.1, 0.9)
    assert np.array_equal(bits(w), bits(w0)) and not np.any(bits(v))


def test_quadratic_convergence():
    # f(w) = 1/2 |w|^2, each of 4 workers pushes g = w (S:220, S:633 corrected
    # per reading R13: with mu=0.9 the norm oscillates, bound only).
    w = values_np(1, 0, 64, 20) + f32(1.0)
    n0 = np.linalg.norm(w)
    v = np.zeros_like(w)
    for _ in range(100):
        w, v, _ = oracle.round_([64], [w] * 4, w, v, 0.1, 0.9)
    assert np.linalg.norm(w) / n0 < 1e-3
    # mu = 0: strictly decreasing until below 1e-6
    w = values_np(1, 0, 64, 20) + f32(1.0)
    v = np.zeros_like(w)
    prev = np.linalg.norm(w)
    while prev > 1e-6:
        w, v, _ = oracle.round_([64], [w] * 4, w, v, 0.1, 0.0)
        cur = np.linalg.norm(w)
        assert cur < prev
        prev = cur


# ------------------------------------------------------ invariances / ref
def test_chunk_size_order_thread_invariance():
    sizes = manifest("tiny")
    grads, w0, v0 = _inputs(sizes, 4)
    base = oracle.round_(sizes, grads, w0, v0, 0.1, 0.9)
    for cb in (4, 12, 4096, 16384, 65536, 1 << 20):
        out = oracle.round_(sizes, grads, w0, v0, 0.1, 0.9, chunk_bytes=cb)
        for a, b in zip(base, out):
            assert np.array_equal(bits(a), bits(b))
    cnt = oracle.chunk_count(sizes, 32768)
    perm = np.random.default_rng(0).permutation(cnt).astype(np.uint32)
    for out in (oracle.round_(sizes, grads, w0, v0, 0.1, 0.9, order=perm),
                oracle.round_(sizes, grads, w0, v0, 0.1, 0.9, nthreads=4)):
        for a, b in zip(base, out):
            assert np.array_equal(bits(a), bits(b))


@pytest.mark.parametrize("N", [1, 2, 3, 4, 7, 8])
def test_numpy_ref_bit_identical(N):
    sizes = [3, 3, 9408, 64, 64, 20000, 1000]
    grads, w0, v0 = _inputs(sizes, N, seed=N)
    a = oracle.round_(sizes, grads, w0, v0, 0.1, 0.9, chunk_bytes=16384)
    b = ref.round_(sizes, grads, w0, v0, 0.1, 0.9, chunk_bytes=16384)
    for x, y in zip(a, b):
        assert np.array_equal(bits(x), bits(y))


def test_rescale_equals_division_for_powers_of_two():
    # reading R2: g = s * (1/N) is bit-identical to s / N when N is a power of 2
    s = values_np(9, 0, 100000, 25) * f32(8)
    for N in (1, 2, 4, 8):
        assert np.array_equal(bits(s * (f32(1) / f32(N))), bits(s / f32(N)))


def test_elems_matches_round():
    sizes = [5000, 77]
    grads, w0, v0 = _inputs(sizes, 8, seed=3)
    w, v, s = oracle.round_(sizes, grads, w0, v0, 0.1, 0.9)
    idx = np.array([0, 1, 4999, 5000, 5076, 1234])
    we, ve, se = oracle.elems(np.stack([g[idx] for g in grads]), w0[idx], v0[idx], 0.1, 0.9)
    assert np.array_equal(bits(we), bits(w[idx]))
    assert np.array_equal(bits(ve), bits(v[idx]))
    assert np.array_equal(bits(se), bits(s[idx]))


@pytest.mark.parametrize("seed", range(12))
def test_random_manifests_two_oracles_agree(seed):
    """Random manifests / chunk sizes / worker counts / hyper-parameters: the
    C oracle and the independent numpy oracle agree bit for bit, and the
    result does not depend on the chunk size."""
    rng = np.random.default_rng(500 + seed)
    K = int(rng.integers(1, 9))
    sizes = [int(x) for x in rng.choice([1, 2, 3, 7, 32, 33, 500, 4096, 9999], K)]
    N = int(rng.integers(1, 10))
    cb = int(rng.choice([4, 12, 64, 4096, 32768]))
    lr = float(rng.choice([0.1, 0.37, 0.0]))
    mu = float(rng.choice([0.9, 0.0, 0.5]))
    grads, w0, v0 = _inputs(sizes, N, seed=seed + 100)
    a = oracle.round_(sizes, grads, w0, v0, lr, mu, chunk_bytes=cb)
    b = ref.round_(sizes, grads, w0, v0, lr, mu, chunk_bytes=cb)
    c = oracle.round_(sizes, grads, w0, v0, lr, mu, chunk_bytes=32768)
    for x, y, z in zip(a, b, c):
        assert np.array_equal(bits(x), bits(y))
        assert np.array_equal(bits(x), bits(z))
