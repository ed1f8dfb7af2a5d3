"""GPU parity: the sm_100a path vs the CPU oracle, through the C ABI (-m gpu).

Inputs are generated independently on each side from the same seeded
counter-based streams (workloads.generate): on the device by fullmant_torch
into the padded layout (padding filled with NaN so any read of padding would
show), on the host by fullmant_np for the oracle.  Nothing the CUDA path
writes is ever fed to the oracle.  The values are FULL-MANTISSA (random 24-bit
significands over 31 binades, both signs), so summing the workers in any
order other than worker-id order changes most results (tests/test_generate.py
pins that, tests/test_gpu_order.py shows the kernels fail it when the order
is wrong): bit-exactness here is evidence of the worker-order sum itself.

Bar (BASELINE.json north_star): chunk table and the worker-order sum
bit-exact; w' and v' within 1e-6 relative -- this build asserts bit-exact for
all three (reading R5: no contraction on either side), and reports
the max relative error when that fails.
"""
import numpy as np
import pytest

import oracle
from workloads import manifest, values_np, grad_stream
from workloads.generate import fullmant_at_np, fullmant_np
from conftest import read_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

f32 = np.float32
DEV = "cuda:0"


def bits(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32)


def assert_bits_equal(got, ref, what):
    got, ref = np.asarray(got, f32), np.asarray(ref, f32)
    if not np.array_equal(bits(got), bits(ref)):
        bad = np.flatnonzero(bits(got) != bits(ref))
        rel = np.max(np.abs(got[bad].astype(np.float64) - ref[bad]) /
                     np.maximum(np.abs(ref[bad].astype(np.float64)), 2.0 ** -126))
        raise AssertionError(f"{what}: {bad.size} of {ref.size} elements differ bitwise, "
                             f"first at {bad[:5]}, max rel err {rel:.3e}")


def _hub(sizes, N, **kw):
    from paper_1805_07891_b200 import PHub
    return PHub(sizes, N, device=0, **kw)


def _pad_index(hub):
    return torch.as_tensor(hub.padded_index(), device=DEV)


def device_grads(hub, N, seed=0):
    """N padded device buffers with full-mantissa stream values at real
    elements, NaN in padding."""
    from workloads.generate import fullmant_torch
    idx = _pad_index(hub)
    out = []
    for w in range(N):
        buf = torch.full((hub.E_padded,), float("nan"), dtype=torch.float32, device=DEV)
        buf[idx] = fullmant_torch(grad_stream(w) + 37 * seed, 0, hub.E, DEV)
        out.append(buf)
    return out


def host_grads(E, N, seed=0):
    return [fullmant_np(grad_stream(w) + 37 * seed, 0, E) for w in range(N)]


def host_state(E, seed=0):
    return fullmant_np(1 + 37 * seed, 0, E), fullmant_np(2 + 37 * seed, 0, E)


def run_round(hub, grads_dev, mode="borrow"):
    for w, g in enumerate(grads_dev):
        hub.push(w, g, mode=mode)
    hub.aggregate_optimize()
    torch.cuda.synchronize()


def check_round(sizes, N, chunk_bytes=32768, kernel=None, seed=0, lr=0.1, mu=0.9, rescale=0.0):
    from paper_1805_07891_b200 import capi
    hub = _hub(sizes, N, chunk_size_bytes=chunk_bytes, keep_aggregate=True, lr=lr, momentum=mu,
               rescale=rescale)
    w0, v0 = host_state(hub.E, seed)
    hub.load_state(w0, v0)
    if kernel is not None:
        hub.set_option(capi.PHUB_OPT_KERNEL, kernel)
    gd = device_grads(hub, N, seed)
    before = hub.kernel_launches
    run_round(hub, gd)
    launches = hub.kernel_launches - before
    w, v, s = hub.read_state()
    rw, rv, rs = oracle.round_(sizes, host_grads(hub.E, N, seed), w0, v0, lr, mu, rescale,
                               chunk_bytes=chunk_bytes)
    assert_bits_equal(s, rs, "sum s")
    assert_bits_equal(v, rv, "momentum v'")
    assert_bits_equal(w, rw, "weights w'")
    return hub, launches


SMALL = [3, 3, 9408, 64, 64, 4096, 20000, 1000, 262144, 7]   # 3-element keys break 16-B alignment


# ------------------------------------------------------------- basic rounds
def test_tiny_config_bit_exact():
    hub, launches = check_round(manifest("tiny"), 4)
    assert launches == 1                      # one fused kernel per round
    assert hub.iteration == 1


@pytest.mark.parametrize("kernel", ["FLAT", "FLAT128", "TILES", "WIDE", "BULK"])
def test_kernel_variants_bit_exact(kernel):
    from paper_1805_07891_b200 import capi
    _, launches = check_round(SMALL, 8, kernel=getattr(capi, f"PHUB_KERNEL_{kernel}"))
    assert launches == (8 if kernel == "WIDE" else 1)


@pytest.mark.parametrize("N", [1, 2, 3, 5, 7, 8, 9, 16, 33])
def test_worker_counts(N):
    check_round(SMALL, N, seed=N)


@pytest.mark.parametrize("N", [1, 3, 8])
@pytest.mark.parametrize("name", ["tiny", "resnet50"])
def test_bulk_kernel_configs(N, name):
    from paper_1805_07891_b200 import capi
    check_round(manifest(name), N, kernel=capi.PHUB_KERNEL_BULK, seed=N)


@pytest.mark.parametrize("cb", [4, 12, 64, 4096, 32768, 1 << 20])
def test_chunk_sizes(cb):
    check_round(SMALL, 4, chunk_bytes=cb)


def test_tiles_small_tile_size():
    from paper_1805_07891_b200 import capi
    hub = _hub(SMALL, 3, keep_aggregate=True)
    hub.set_option(capi.PHUB_OPT_TILE_ELEMS, 100)       # ragged tiles inside chunks
    hub.set_option(capi.PHUB_OPT_KERNEL, capi.PHUB_KERNEL_TILES)
    w0, v0 = host_state(hub.E)
    hub.load_state(w0, v0)
    run_round(hub, device_grads(hub, 3))
    w, v, s = hub.read_state()
    rw, rv, rs = oracle.round_(SMALL, host_grads(hub.E, 3), w0, v0, 0.1, 0.9)
    assert_bits_equal(w, rw, "w")
    assert_bits_equal(s, rs, "s")


def test_rescale_and_hyperparameters():
    check_round(SMALL, 3, lr=0.37, mu=0.5, rescale=0.25)
    check_round(SMALL, 6, lr=1e-3, mu=0.0)


# ---------------------------------------------------- push / pull semantics
def test_per_key_and_copy_pushes():
    sizes = SMALL
    N = 4
    hub = _hub(sizes, N, keep_aggregate=True)
    w0, v0 = host_state(hub.E)
    hub.load_state(w0, v0)
    hg = host_grads(hub.E, N)
    starts = np.concatenate([[0], np.cumsum(sizes)])
    # worker 0: per-key BORROW of unpadded device slices (own allocations)
    keep = []
    for k, nk in enumerate(sizes):
        t = torch.tensor(hg[0][starts[k]:starts[k + 1]], device=DEV)
        keep.append(t)
        hub.push(0, t, key=k, mode="borrow")
    # worker 1: whole-model COPY from a padded host buffer
    pad = np.full(hub.E_padded, np.nan, f32)
    pad[hub.padded_index()] = hg[1]
    hub.push(1, pad, mode="copy")
    # worker 2: per-key COPY from host, in reverse key order
    for k in reversed(range(len(sizes))):
        hub.push(2, np.ascontiguousarray(hg[2][starts[k]:starts[k + 1]]), key=k, mode="copy")
    # worker 3: whole-model BORROW (device, padded)
    d3 = device_grads(hub, 4)[3]
    hub.push(3, d3, mode="borrow")
    hub.aggregate_optimize()
    w, v, s = hub.read_state()
    rw, rv, rs = oracle.round_(sizes, hg, w0, v0, 0.1, 0.9)
    assert_bits_equal(s, rs, "s")
    assert_bits_equal(w, rw, "w")
    assert_bits_equal(v, rv, "v")


def test_errors_leave_state_unchanged():
    from paper_1805_07891_b200 import PhubError, capi
    sizes = SMALL
    hub = _hub(sizes, 2, keep_aggregate=True)
    w0, v0 = host_state(hub.E)
    hub.load_state(w0, v0)
    gd = device_grads(hub, 2)

    def status(fn):
        with pytest.raises(PhubError) as e:
            fn()
        return capi.STATUS_NAMES[e.value.status]

    assert status(lambda: hub.aggregate_optimize()) == "PHUB_ERR_INCOMPLETE"
    hub.push(0, gd[0])
    assert status(lambda: hub.push(0, gd[0])) == "PHUB_ERR_DUPLICATE_PUSH"
    assert status(lambda: hub.push(0, gd[0][:sizes[1]], key=1)) == "PHUB_ERR_DUPLICATE_PUSH"
    assert status(lambda: hub.push(2, gd[1])) == "PHUB_ERR_BAD_WORKER"
    assert status(lambda: hub.push(1, gd[1], key=len(sizes))) == "PHUB_ERR_BAD_KEY"
    assert status(lambda: hub.push(1, gd[1][:5], key=0)) == "PHUB_ERR_LENGTH_MISMATCH"
    assert status(lambda: hub.push(1, gd[1][: hub.E_padded - 32])) == "PHUB_ERR_LENGTH_MISMATCH"
    assert status(lambda: hub.push(1, np.zeros(hub.E_padded, f32), mode="borrow")) == \
        "PHUB_ERR_INVALID_ARGUMENT"                                   # host ptr cannot be borrowed
    assert status(lambda: hub.push(1, gd[1][1:], n=hub.E_padded - 1)) == "PHUB_ERR_LENGTH_MISMATCH"
    assert status(lambda: hub.push(1, gd[1][1:1 + sizes[0]], key=0)) == \
        "PHUB_ERR_INVALID_ARGUMENT"                                   # BORROW needs 16-B alignment
    assert status(lambda: hub.aggregate_optimize()) == "PHUB_ERR_INCOMPLETE"
    assert hub.iteration == 0
    hub.push(1, gd[1])
    hub.aggregate_optimize()
    w, v, s = hub.read_state()
    rw, rv, rs = oracle.round_(sizes, host_grads(hub.E, 2), w0, v0, 0.1, 0.9)
    assert_bits_equal(w, rw, "w after recovered round")
    assert hub.iteration == 1


def test_pull_semantics():
    sizes = SMALL
    init = fullmant_np(5, 0, sum(sizes))
    hub = _hub(sizes, 3, init_weights=init)
    starts = np.concatenate([[0], np.cumsum(sizes)])
    dst = np.empty(sizes[2], f32)
    hub.pull(dst, key=2)
    torch.cuda.synchronize()
    assert_bits_equal(dst, init[starts[2]:starts[3]], "pull before aggregate (S:365)")
    gd = device_grads(hub, 3)
    run_round(hub, gd)
    rw, _, _ = oracle.round_(sizes, host_grads(hub.E, 3), init, np.zeros_like(init), 0.1, 0.9)
    full = np.empty(hub.E_padded, f32)
    hub.pull(full)                                   # host destination
    torch.cuda.synchronize()
    assert_bits_equal(full[hub.padded_index()], rw, "ALL_KEYS pull")
    for k in (0, 6, 9):
        d = torch.empty(sizes[k], device=DEV)
        hub.pull(d, key=k)                           # device destination
        torch.cuda.synchronize()
        assert_bits_equal(d.cpu().numpy(), rw[starts[k]:starts[k + 1]], f"pull key {k}")
    wv = hub.weights()                               # zero-copy pull
    assert_bits_equal(wv.cpu().numpy()[hub.padded_index()], rw, "zero-copy weights")


def test_pushpull():
    sizes = SMALL
    hub = _hub(sizes, 3)
    gd = device_grads(hub, 3)
    out = torch.empty(hub.E_padded, device=DEV)
    for w in range(3):
        hub.pushpull(w, gd[w], dst=out)
        assert hub.iteration == (1 if w == 2 else 0)
    torch.cuda.synchronize()
    rw, _, _ = oracle.round_(sizes, host_grads(hub.E, 3), np.zeros(hub.E, f32),
                             np.zeros(hub.E, f32), 0.1, 0.9)
    assert_bits_equal(out.cpu().numpy()[hub.padded_index()], rw, "pushpull result")


def test_multi_round():
    sizes = SMALL
    N = 4
    hub = _hub(sizes, N, keep_aggregate=True)
    w, v = host_state(hub.E, 1)
    hub.load_state(w, v)
    for r in range(3):
        run_round(hub, device_grads(hub, N, seed=r))
        w, v, _ = oracle.round_(sizes, host_grads(hub.E, N, seed=r), w, v, 0.1, 0.9)
    gw, gv, _ = hub.read_state()
    assert_bits_equal(gw, w, "w after 3 rounds")
    assert_bits_equal(gv, v, "v after 3 rounds")
    assert hub.iteration == 3


# -------------------------------------------------------- special cases
@pytest.mark.parametrize("row", read_golden("nag_cases.txt"), ids=lambda r: r[0])
def test_nag_golden_on_gpu(row):
    name, _cite, N, lr, mu, resc, w0, v0, g, ew, ev = row
    N = int(N)
    vals = [1.0, 3.0] if name == "s175" else [float(g)] * N
    hub = _hub([1], N, lr=float(lr), momentum=float(mu), rescale=float(resc),
               init_weights=np.array([float(w0)], f32))
    hub.load_state(None, np.array([float(v0)], f32))
    bufs = []
    for w in range(N):
        b = torch.zeros(hub.E_padded, device=DEV)
        b[0] = vals[w]
        bufs.append(b)
    run_round(hub, bufs)
    gw, gv, _ = hub.read_state()
    assert bits(gw)[0] == int(ew, 16) and bits(gv)[0] == int(ev, 16)


def test_signed_zero_and_dyadic():
    from workloads import dyadic_np
    sizes = [5, 1000, 3]
    hub = _hub(sizes, 8, keep_aggregate=True)
    idx = _pad_index(hub)
    zs = []
    for w in range(8):
        b = torch.full((hub.E_padded,), float("nan"), device=DEV)
        b[idx] = -0.0
        zs.append(b)
    run_round(hub, zs)
    _, _, s = hub.read_state()
    assert not np.any(bits(s))                       # +0 start: never -0 (reading R4)
    hg = [dyadic_np(60 + w, hub.E) for w in range(8)]
    bufs = []
    for w in range(8):
        b = torch.full((hub.E_padded,), float("nan"), device=DEV)
        b[idx] = torch.tensor(hg[w], device=DEV)
        bufs.append(b)
    run_round(hub, bufs)
    _, _, s = hub.read_state()
    exact = np.sum(np.stack(hg).astype(np.float64), axis=0)
    assert np.array_equal(s.astype(np.float64), exact)


def test_lr0_identity():
    sizes = SMALL
    hub = _hub(sizes, 5, lr=0.0)
    w0, v0 = host_state(hub.E, 4)
    hub.load_state(w0, v0)
    run_round(hub, device_grads(hub, 5, seed=4))
    w, _, _ = hub.read_state()
    assert_bits_equal(w, w0, "lr=0 identity")


# ----------------------------------------- owner sharding on one GPU (M2)
@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("policy", ["contig", "lpt"])
def test_owner_sharding_invariance(G, policy):
    sizes = manifest("resnet50")
    N = 4
    E = sum(sizes)
    w0, v0 = host_state(E, 2)
    rw, rv, rs = oracle.round_(sizes, host_grads(E, N, 2), w0, v0, 0.1, 0.9)
    got_w = np.full(E, np.nan, f32)
    got_v = np.full(E, np.nan, f32)
    gd = None
    starts = np.concatenate([[0], np.cumsum(sizes)])
    for r in range(G):
        hub = _hub(sizes, N, num_owners=G, owner_rank=r, owner_policy=policy)
        hub.load_state(w0, v0)
        if gd is None:
            gd = device_grads(hub, N, 2)
        run_round(hub, gd)
        w, v, _ = hub.read_state()
        tab = hub.chunk_table()
        for k, off, ln, own in zip(tab["key_id"], tab["offset"], tab["length"], tab["owner"]):
            if own == r:
                a = int(starts[k] + off)
                got_w[a:a + int(ln)] = w[a:a + int(ln)]
                got_v[a:a + int(ln)] = v[a:a + int(ln)]
        hub.close()
    assert_bits_equal(got_w, rw, f"w' union over {G} owners ({policy})")
    assert_bits_equal(got_v, rv, f"v' union over {G} owners ({policy})")


def test_chunk_table_matches_oracle():
    for name in ("tiny", "resnet269"):
        m = manifest(name)
        for G, pol in ((1, "contig"), (4, "lpt"), (8, "contig")):
            hub = _hub(m, 2, num_owners=G, owner_rank=G - 1, owner_policy=pol)
            t = hub.chunk_table()
            ref = oracle.chunk_plan(m)
            own = np.zeros(len(ref["length"]), np.int32) if G == 1 else \
                (oracle.owners_lpt if pol == "lpt" else oracle.owners_contig)(ref["length"], G)
            assert oracle.canonical_text(t, t["owner"]) == oracle.canonical_text(ref, own)
            hub.close()


# ------------------------------ full BASELINE sizes, sampled outputs
def _sample_indices(sizes, chunk_bytes, rng, n_random=20000):
    E = sum(sizes)
    starts = np.concatenate([[0], np.cumsum(sizes)])
    ce = chunk_bytes // 4
    pts = [rng.integers(0, E, n_random)]
    pts.append(starts[:-1])                                  # key starts
    pts.append(starts[1:] - 1)                               # key ends
    for k in range(len(sizes)):                              # chunk boundaries
        b = np.arange(starts[k], starts[k + 1], ce)
        pts.append(b[:64])
        pts.append(np.maximum(b[:64] - 1, starts[k]))
    return np.unique(np.concatenate(pts)).astype(np.int64)


@pytest.mark.parametrize("name,N,cb", [
    ("resnet50", 8, 32768), ("alexnet", 8, 32768), ("vgg19", 8, 32768),
    *[("resnet269", 8, 4096 << i) for i in range(9)],        # BJ configs[4] sweep
])
def test_full_size_sampled(name, N, cb):
    from workloads.generate import fullmant_torch
    sizes = manifest(name)
    hub = _hub(sizes, N, chunk_size_bytes=cb)                # bench launch config (AUTO)
    E = hub.E
    idx_pad = _pad_index(hub)
    w0 = fullmant_torch(1, 0, E, DEV)
    v0 = fullmant_torch(2, 0, E, DEV)
    hub.load_state(w0, v0)
    del w0, v0
    gd = []
    for w in range(N):
        b = torch.full((hub.E_padded,), float("nan"), device=DEV)
        b[idx_pad] = fullmant_torch(grad_stream(w), 0, E, DEV)
        gd.append(b)
    run_round(hub, gd)
    del gd
    rng = np.random.default_rng(len(sizes) * 7919 + cb)
    samp = _sample_indices(sizes, cb, rng)
    w_all, v_all, _ = hub.read_state()
    # oracle on independently generated inputs at the sampled elements
    g = np.stack([fullmant_at_np(grad_stream(w), samp) for w in range(N)])
    rw, rv, _ = oracle.elems(g, fullmant_at_np(1, samp), fullmant_at_np(2, samp), 0.1, 0.9)
    assert_bits_equal(w_all[samp], rw, f"{name}@{cb} sampled w'")
    assert_bits_equal(v_all[samp], rv, f"{name}@{cb} sampled v'")
    hub.close()


# -------------------------------------------- fused replica stores (P2P pull)
def test_replica_stores_single_gpu():
    """The fused pull path (phub_set_replicas) stores w' of the owned range into
    extra replicas; on one GPU local buffers stand in for peer replicas."""
    from paper_1805_07891_b200 import capi
    sizes = manifest("resnet50")
    G, N = 4, 4
    E = sum(sizes)
    w0, v0 = host_state(E, 3)
    rw, _, _ = oracle.round_(sizes, host_grads(E, N, 3), w0, v0, 0.1, 0.9)
    reps = None
    gd = None
    for r in range(G):
        hub = _hub(sizes, N, num_owners=G, owner_rank=r, owner_policy="contig")
        hub.load_state(w0, v0)
        if reps is None:
            reps = [torch.full((hub.E_padded,), float("nan"), device=DEV) for _ in range(2)]
            gd = device_grads(hub, N, 3)
        capi.phub_set_replicas(hub.ctx, [t.data_ptr() for t in reps])
        run_round(hub, gd)
        hub.close()
    from paper_1805_07891_b200 import PHub
    h = PHub(sizes, N, device=0)
    pidx = h.padded_index()
    h.close()
    for t in reps:
        assert_bits_equal(t.cpu().numpy()[pidx], rw, "replica assembled from 4 owners")


def test_replica_errors():
    from paper_1805_07891_b200 import PhubError, capi
    hub = _hub(SMALL, 2, num_owners=2, owner_rank=0, owner_policy="lpt")
    t = torch.zeros(hub.E_padded, device=DEV)
    with pytest.raises(PhubError):
        capi.phub_set_replicas(hub.ctx, [t.data_ptr()])              # LPT: no contiguous range
    hub.close()
    hub = _hub(SMALL, 2)
    with pytest.raises(PhubError):
        capi.phub_set_replicas(hub.ctx, [t.data_ptr() + 4])          # misaligned
    with pytest.raises(PhubError):
        capi.phub_set_replicas(hub.ctx, [np.zeros(4, f32).ctypes.data])   # host memory
    capi.phub_set_replicas(hub.ctx, [t.data_ptr()])
    hub.set_option(capi.PHUB_OPT_KERNEL, capi.PHUB_KERNEL_TILES)
    for w, g in enumerate(device_grads(hub, 2)):
        hub.push(w, g)
    with pytest.raises(PhubError) as e:
        hub.aggregate_optimize()                                        # replicas need flat
    assert capi.STATUS_NAMES[e.value.status] == "PHUB_ERR_UNSUPPORTED"
    hub.close()


def test_shared_alloc_and_ipc_handle():
    from paper_1805_07891_b200 import capi
    p = capi.phub_alloc_shared(0, 1 << 20)
    h = capi.phub_ipc_get_handle(0, p)
    assert len(h) == 64 and any(h)
    capi.phub_free_shared(0, p)


# ------------------------------------------- streaming aggregation (NEXT-1)
def test_streaming_aggregate_ready_backward_order():
    """Keys arrive in reverse order (a backward pass); each key is aggregated as
    soon as all N workers pushed it.  Same bits as one round."""
    sizes = SMALL
    N = 3
    hub = _hub(sizes, N, keep_aggregate=True)
    w0, v0 = host_state(hub.E, 5)
    hub.load_state(w0, v0)
    hg = host_grads(hub.E, N, 5)
    starts = np.concatenate([[0], np.cumsum(sizes)])
    keep = []
    total = 0
    for k in reversed(range(len(sizes))):
        for w in range(N):
            t = torch.tensor(hg[w][starts[k]:starts[k + 1]], device=DEV)
            keep.append(t)
            hub.push(w, t, key=k)
            if w < N - 1:
                assert hub.aggregate_ready() == 0        # not all workers yet
        total += hub.aggregate_ready()
        assert hub.iteration == (1 if k == 0 else 0)
    assert total == len(sizes)
    torch.cuda.synchronize()
    w, v, s = hub.read_state()
    rw, rv, rs = oracle.round_(sizes, hg, w0, v0, 0.1, 0.9)
    assert_bits_equal(s, rs, "streamed s")
    assert_bits_equal(w, rw, "streamed w")
    assert_bits_equal(v, rv, "streamed v")


def test_streaming_then_aggregate_rest():
    sizes = SMALL
    N = 2
    hub = _hub(sizes, N)
    w0, v0 = host_state(hub.E, 6)
    hub.load_state(w0, v0)
    gd = device_grads(hub, N, 6)
    hg = host_grads(hub.E, N, 6)
    starts = np.concatenate([[0], np.cumsum(sizes)])
    keep = []
    for k in (2, 3, 7):                                   # a few keys stream early
        for w in range(N):
            t = torch.tensor(hg[w][starts[k]:starts[k + 1]], device=DEV)
            keep.append(t)
            hub.push(w, t, key=k)
    assert hub.aggregate_ready() == 3
    for k in range(len(sizes)):
        if k in (2, 3, 7):
            continue
        for w in range(N):
            t = torch.tensor(hg[w][starts[k]:starts[k + 1]], device=DEV)
            keep.append(t)
            hub.push(w, t, key=k)
    hub.aggregate_optimize()                              # only the remaining keys
    assert hub.iteration == 1
    w, v, _ = hub.read_state()
    rw, rv, _ = oracle.round_(sizes, hg, w0, v0, 0.1, 0.9)
    assert_bits_equal(w, rw, "w")
    assert_bits_equal(v, rv, "v")
    # the next iteration starts clean: whole-model pushes, flat kernel
    run_round(hub, gd)
    w2, _, _ = hub.read_state()
    rw2, _, _ = oracle.round_(sizes, hg, rw, rv, 0.1, 0.9)
    assert_bits_equal(w2, rw2, "w after next round")


def test_copy_push_two_slots_pipelined():
    """COPY pushes alternate between two receive slots, so round k+1's H2D
    copies may overlap round k's kernel (the bench's e2e pipeline)."""
    sizes = SMALL
    N = 3
    hub = _hub(sizes, N)
    w, v = host_state(hub.E, 7)
    hub.load_state(w, v)
    pidx = hub.padded_index()
    s_in, s_c = torch.cuda.Stream(), torch.cuda.Stream()
    ev_c = []
    host = []
    for r in range(4):
        hg = host_grads(hub.E, N, 10 + r)
        bufs = []
        for g in hg:
            h = torch.full((hub.E_padded,), float("nan"), pin_memory=True)
            h.numpy()[pidx] = g
            bufs.append(h)
        host.append(bufs)
        if r >= 2:
            s_in.wait_event(ev_c[r - 2])
        for k, h in enumerate(bufs):
            hub.push(k, h, mode="copy", stream=s_in)
        e_in = torch.cuda.Event()
        e_in.record(s_in)
        s_c.wait_event(e_in)
        hub.aggregate_optimize(stream=s_c)
        e = torch.cuda.Event()
        e.record(s_c)
        ev_c.append(e)
        w, v, _ = oracle.round_(sizes, hg, w, v, 0.1, 0.9)
    torch.cuda.synchronize()
    gw, gv, _ = hub.read_state()
    assert_bits_equal(gw, w, "w after 4 pipelined COPY rounds")
    assert_bits_equal(gv, v, "v after 4 pipelined COPY rounds")


# ----------------------------------------------- chained-exchange building blocks
def test_partial_sum_and_range_aggregate_chain_on_one_gpu():
    """The chained exchange on one GPU: a partial sum of workers 0..2 (as a
    previous rank would store it), then a context with N' = 1 + 3 workers
    (the partial + workers 3..5, rescale 1/6) aggregated piece by piece --
    bit-identical to the 6-worker oracle round."""
    from paper_1805_07891_b200 import PHub, capi
    sizes = manifest("resnet50")
    E = sum(sizes)
    w0, v0 = host_state(E, 8)
    head = _hub(sizes, 3)
    gd = device_grads(head, 6, 8)
    for g in gd:
        g.nan_to_num_(0.0)                  # padding must be finite for the flat partial sum
    part = torch.empty(head.E_padded, device=DEV)
    capi.phub_partial_sum(head.ctx, [g.data_ptr() for g in gd[:3]], part.data_ptr(), 0,
                          head.E_padded, head._stream(None))
    tail = PHub(sizes, 4, device=0, rescale=1.0 / 6)
    tail.load_state(w0, v0)
    tail.push(0, part)
    for k in range(3):
        tail.push(1 + k, gd[3 + k])
    Ep = tail.E_padded
    cuts = [0, 4096, 4096 * 9, Ep // 2 // 64 * 64, Ep]
    for b, e in zip(cuts[:-1], cuts[1:]):
        assert tail.iteration == 0
        capi.phub_aggregate_range(tail.ctx, b, e, tail._stream(None))
    assert tail.iteration == 1
    torch.cuda.synchronize()
    w, v, _ = tail.read_state()
    rw, rv, _ = oracle.round_(sizes, host_grads(E, 6, 8), w0, v0, 0.1, 0.9)
    assert_bits_equal(w, rw, "chained w")
    assert_bits_equal(v, rv, "chained v")
    head.close()
    tail.close()


def test_range_aggregate_order_errors():
    from paper_1805_07891_b200 import PhubError, capi
    hub = _hub(SMALL, 2)
    gd = device_grads(hub, 2)
    for w, g in enumerate(gd):
        hub.push(w, g)
    with pytest.raises(PhubError):
        capi.phub_aggregate_range(hub.ctx, 64, 128, 0)          # must start at the range begin
    capi.phub_aggregate_range(hub.ctx, 0, 64, 0)
    with pytest.raises(PhubError):
        hub.aggregate_optimize()                                # iteration is being ranged
    capi.phub_aggregate_range(hub.ctx, 64, hub.E_padded, 0)
    assert hub.iteration == 1
    hub.close()


def test_stage_flags_signal_and_bounded_wait():
    """phub_sync: a partial sum raises a flag that a range aggregate waits on;
    a wait on a flag nobody raises gives up (bounded) and is counted."""
    from paper_1805_07891_b200 import PHub, capi
    sizes = manifest("tiny")
    E = sum(sizes)
    head = _hub(sizes, 2)
    gd = [g.nan_to_num_(0.0) for g in device_grads(head, 4, 9)]
    flags = torch.zeros(4, dtype=torch.int32, device=DEV)
    part = torch.empty(head.E_padded, device=DEV)
    st = head._stream(None)
    capi.phub_partial_sum(head.ctx, [g.data_ptr() for g in gd[:2]], part.data_ptr(), 0,
                          head.E_padded, st, signal=(flags.data_ptr(), 7))
    tail = PHub(sizes, 3, device=0, rescale=0.25)
    w0, v0 = host_state(E, 9)
    tail.load_state(w0, v0)
    tail.push(0, part)
    tail.push(1, gd[2])
    tail.push(2, gd[3])
    capi.phub_aggregate_range(tail.ctx, 0, tail.E_padded, st, wait=(flags.data_ptr(), 7))
    torch.cuda.synchronize()
    assert int(flags[0].item()) == 7
    assert capi.phub_sync_timeouts(tail.ctx) == 0
    w, _, _ = tail.read_state()
    rw, _, _ = oracle.round_(sizes, host_grads(E, 4, 9), w0, v0, 0.1, 0.9)
    assert_bits_equal(w, rw, "flag-ordered chain on one GPU")
    # a flag that is never raised: the wait expires (~2 s), the work is skipped, and
    # the context turns sticky-failed: the NEXT call reports it, never a stale w'
    for k in range(3):
        tail.push(k, gd[k])
    capi.phub_aggregate_range(tail.ctx, 0, tail.E_padded, st, wait=(flags.data_ptr() + 4, 1))
    torch.cuda.synchronize()
    assert capi.phub_sync_timeouts(tail.ctx) >= 1
    assert_sticky_timeout(tail, gd)
    head.close()
    tail.close()


def assert_sticky_timeout(hub, gd):
    """After an expired device wait every data call on the context fails with
    PHUB_ERR_SYNC_TIMEOUT (header conventions)."""
    from paper_1805_07891_b200 import PhubError, capi

    def status(fn):
        with pytest.raises(PhubError) as e:
            fn()
        return capi.STATUS_NAMES[e.value.status]

    assert capi.STATUS_NAMES[capi.phub_check(hub.ctx)] == "PHUB_ERR_SYNC_TIMEOUT"
    assert status(lambda: hub.push(0, gd[0])) == "PHUB_ERR_SYNC_TIMEOUT"
    assert status(lambda: hub.read_state()) == "PHUB_ERR_SYNC_TIMEOUT"
    assert status(lambda: hub.pull(torch.empty(hub.E_padded, device=DEV))) == \
        "PHUB_ERR_SYNC_TIMEOUT"
    assert status(lambda: hub.weights_ptr()) == "PHUB_ERR_SYNC_TIMEOUT"
    assert status(lambda: hub.synchronize()) == "PHUB_ERR_SYNC_TIMEOUT"


@pytest.mark.parametrize("block", [2048, 12288, 16384, 32768])
def test_block_streaming_flags_chain_on_one_gpu(block):
    """phub_sync block form: a partial sum raises one flag per block and a
    range aggregate waits on them block by block (same stream here: the
    producer finishes first; tests/test_gpu_emulated_ranks.py runs them
    concurrently) -- bit-identical to the 6-worker oracle round; every flag
    raised exactly to the epoch; a bad block size is refused; an unraised
    flag times out and makes the context sticky-failed."""
    from paper_1805_07891_b200 import PHub, PhubError, capi
    sizes = manifest("resnet50")
    E = sum(sizes)
    w0, v0 = host_state(E, 12)
    head = _hub(sizes, 3)
    gd = device_grads(head, 6, 12)
    Ep = head.E_padded
    nblk = -(-Ep // block)
    flags = torch.zeros(nblk + 1, dtype=torch.int32, device=DEV)
    part = torch.empty(Ep, device=DEV)
    st = head._stream(None)
    with pytest.raises(PhubError):
        capi.phub_partial_sum(head.ctx, [g.data_ptr() for g in gd[:3]], part.data_ptr(), 0, Ep,
                              st, signal=(flags.data_ptr(), 3), block=1000)
    capi.phub_partial_sum(head.ctx, [g.data_ptr() for g in gd[:3]], part.data_ptr(), 0, Ep, st,
                          signal=(flags.data_ptr(), 3), block=block)
    tail = PHub(sizes, 4, device=0, rescale=1.0 / 6, keep_aggregate=True)
    tail.load_state(w0, v0)
    tail.push(0, part)
    for k in range(3):
        tail.push(1 + k, gd[3 + k])
    capi.phub_aggregate_range(tail.ctx, 0, Ep, st, wait=(flags.data_ptr(), 3), block=block)
    torch.cuda.synchronize()
    assert tail.iteration == 1
    f = flags.cpu().numpy()
    assert (f[:nblk] == 3).all() and f[nblk] == 0
    assert capi.phub_sync_timeouts(tail.ctx) == 0
    w, v, s = tail.read_state()
    rw, rv, rs = oracle.round_(sizes, host_grads(E, 6, 12), w0, v0, 0.1, 0.9)
    assert_bits_equal(s, rs, "block-streamed aggregate")
    assert_bits_equal(w, rw, "block-streamed w")
    assert_bits_equal(v, rv, "block-streamed v")
    # flags never raised for epoch 4: the waits expire once (~2 s), the work is skipped
    for k in range(4):
        tail.push(k, gd[k])
    capi.phub_aggregate_range(tail.ctx, 0, Ep, st, wait=(flags.data_ptr(), 4), block=block)
    torch.cuda.synchronize()
    assert capi.phub_sync_timeouts(tail.ctx) >= 1
    assert_sticky_timeout(tail, gd)
    head.close()
    tail.close()


def test_removed_push_mode_is_refused():
    """Round 2 removed PHUB_CONSUME (mode 2): it is an invalid mode now."""
    from paper_1805_07891_b200 import PhubError, capi
    hub = _hub(SMALL, 2)
    gd = device_grads(hub, 1)
    with pytest.raises(PhubError) as e:
        capi.phub_push(hub.ctx, 0, capi.PHUB_ALL_KEYS, gd[0].data_ptr(), hub.E_padded, 2, 0)
    assert capi.STATUS_NAMES[e.value.status] == "PHUB_ERR_INVALID_ARGUMENT"
    hub.close()


def test_push_batch_per_key_and_all_or_nothing():
    from paper_1805_07891_b200 import PhubError, capi
    sizes = SMALL
    N = 3
    hub = _hub(sizes, N, keep_aggregate=True)
    w0, v0 = host_state(hub.E, 11)
    hub.load_state(w0, v0)
    hg = host_grads(hub.E, N, 11)
    starts = np.concatenate([[0], np.cumsum(sizes)])
    keys = [[torch.tensor(hg[w][starts[k]:starts[k + 1]], device=DEV) for k in range(len(sizes))]
            for w in range(N)]
    # a batch with a duplicate inside it is rejected whole
    with pytest.raises(PhubError) as e:
        hub.push_batch([(0, 0, keys[0][0]), (1, 0, keys[1][0]), (0, 0, keys[0][0])])
    assert capi.STATUS_NAMES[e.value.status] == "PHUB_ERR_DUPLICATE_PUSH"
    # a bad length late in the batch rolls back the earlier entries
    with pytest.raises(PhubError):
        hub.push_batch([(0, 0, keys[0][0]), (0, 1, keys[0][2])])
    entries = [(w, k, keys[w][k]) for k in reversed(range(len(sizes))) for w in range(N)]
    hub.push_batch(entries)                                 # nothing was recorded before
    hub.aggregate_optimize()
    w, v, s = hub.read_state()
    rw, rv, rs = oracle.round_(sizes, hg, w0, v0, 0.1, 0.9)
    assert_bits_equal(s, rs, "batch s")
    assert_bits_equal(w, rw, "batch w")


def test_two_contexts_multi_tenant():
    """Two jobs with separate key namespaces share one GPU."""
    a = _hub(manifest("tiny"), 4)
    b = _hub(SMALL, 3, lr=0.05, momentum=0.5)
    wa, va = host_state(a.E, 12)
    wb, vb = host_state(b.E, 13)
    a.load_state(wa, va)
    b.load_state(wb, vb)
    ga, gb = device_grads(a, 4, 12), device_grads(b, 3, 13)
    for r in range(2):
        for i in range(4):
            a.push(i, ga[i])
            if i < 3:
                b.push(i, gb[i])
        b.aggregate_optimize()
        a.aggregate_optimize()
        wa, va, _ = oracle.round_(manifest("tiny"), host_grads(a.E, 4, 12), wa, va, 0.1, 0.9)
        wb, vb, _ = oracle.round_(SMALL, host_grads(b.E, 3, 13), wb, vb, 0.05, 0.5)
    assert_bits_equal(a.read_state()[0], wa, "tenant a")
    assert_bits_equal(b.read_state()[0], wb, "tenant b")


# ------------------------------------------------------------ randomized
@pytest.mark.parametrize("seed", range(24))
def test_randomized_configs(seed):
    """Random manifests (incl. 1-3 element keys), chunk sizes, worker counts,
    kernels and push modes (whole-model / per-key / COPY / BORROW mixed per
    worker), two rounds -- always bit-exact against the oracle."""
    from paper_1805_07891_b200 import capi
    rng = np.random.default_rng(1000 + seed)
    K = int(rng.integers(1, 12))
    sizes = [int(x) for x in rng.choice([1, 2, 3, 5, 31, 32, 33, 1000, 4096, 9999, 40000], K)]
    cb = int(rng.choice([4, 8, 16, 100, 1024, 4096, 32768, 65536]))
    N = int(rng.integers(1, 13))
    kern = int(rng.choice([capi.PHUB_KERNEL_AUTO, capi.PHUB_KERNEL_TILES]))
    lr = float(rng.choice([0.1, 0.01, 0.0]))
    mu = float(rng.choice([0.9, 0.0, 0.5]))
    hub = _hub(sizes, N, chunk_size_bytes=cb, keep_aggregate=True, lr=lr, momentum=mu)
    E = hub.E
    w, v = host_state(E, 20 + seed)
    hub.load_state(w, v)
    hub.set_option(capi.PHUB_OPT_KERNEL, kern)
    starts = np.concatenate([[0], np.cumsum(sizes)])
    pidx = hub.padded_index()
    keep = []
    for r in range(2):
        hg = host_grads(E, N, 40 + seed * 3 + r)
        for wk in range(N):
            how = int(rng.integers(0, 4))
            if how == 0:                                   # whole model, device, BORROW
                t = torch.full((hub.E_padded,), float("nan"), device=DEV)
                t[torch.as_tensor(pidx, device=DEV)] = torch.as_tensor(hg[wk], device=DEV)
                keep.append(t)
                hub.push(wk, t)
            elif how == 1:                                 # whole model, host, COPY
                h = np.full(hub.E_padded, np.nan, np.float32)
                h[pidx] = hg[wk]
                hub.push(wk, h, mode="copy")
            elif how == 2:                                 # per key, device, BORROW
                for k in rng.permutation(K):
                    t = torch.as_tensor(np.ascontiguousarray(hg[wk][starts[k]:starts[k + 1]]),
                                        device=DEV)
                    keep.append(t)
                    hub.push(wk, t, key=int(k))
            else:                                          # per key, host, COPY
                for k in rng.permutation(K):
                    hub.push(wk, np.ascontiguousarray(hg[wk][starts[k]:starts[k + 1]]),
                             key=int(k), mode="copy")
        hub.aggregate_optimize()
        torch.cuda.synchronize()
        keep.clear()
        w, v, s = oracle.round_(sizes, hg, w, v, lr, mu, chunk_bytes=cb)
    gw, gv, gs = hub.read_state()
    assert_bits_equal(gs, s, f"seed {seed} s")
    assert_bits_equal(gv, v, f"seed {seed} v")
    assert_bits_equal(gw, w, f"seed {seed} w")


def test_hier_exchange_single_rack_and_validation():
    """phub_hier_exchange with one rack (no peers) is the flat round of its P
    workers (oracle.hier_round with R = 1); bad arguments are refused with
    the state unchanged."""
    from paper_1805_07891_b200 import PhubError, capi
    sizes = manifest("resnet50")
    P = 8
    hub = _hub(sizes, P, keep_aggregate=True)
    w0, v0 = host_state(hub.E, 14)
    hub.load_state(w0, v0)
    gd = device_grads(hub, P, 14)
    with pytest.raises(PhubError):                         # nothing pushed yet
        capi.phub_hier_exchange(hub.ctx, 1, 16384, None, None, 0, None, 1)
    for k, g in enumerate(gd):
        hub.push(k, g)
    for bad in [dict(R=2), dict(block=1000), dict(epoch=0)]:
        with pytest.raises(PhubError):
            capi.phub_hier_exchange(hub.ctx, bad.get("R", 1), bad.get("block", 16384), None, None,
                                    0, None, bad.get("epoch", 1))
    assert hub.iteration == 0
    for epoch in (1, 2):
        if epoch == 2:
            for k, g in enumerate(gd):
                hub.push(k, g)
        capi.phub_hier_exchange(hub.ctx, 1, 16384, None, None, 0, None, epoch)
    torch.cuda.synchronize()
    assert hub.iteration == 2
    w, v, s = hub.read_state()
    hg = host_grads(hub.E, P, 14)
    rw, rv, _ = oracle.hier_round(sizes, [hg], w0, v0, 0.1, 0.9)
    rw, rv, rs = oracle.hier_round(sizes, [hg], rw, rv, 0.1, 0.9)
    assert_bits_equal(s, rs, "single-rack hierarchical aggregate")
    assert_bits_equal(w, rw, "single-rack hierarchical w")
    assert_bits_equal(v, rv, "single-rack hierarchical v")
    hub.close()


def test_hier_exchange_rejects_bad_peer_pointers():
    """phub_hier_exchange validates its peer tables on the host before any
    launch: missing or misaligned inbox / flag pointers are refused and the
    iteration is left untouched (a 2-owner context on one GPU, never launched)."""
    from paper_1805_07891_b200 import PHub, PhubError, capi
    sizes = manifest("tiny")
    hub = PHub(sizes, 2, device=0, num_owners=2, owner_rank=0, owner_policy="contig")
    gd = device_grads(hub, 2, 15)
    for k, g in enumerate(gd):
        hub.push(k, g)
    buf = torch.zeros(1 << 16, device=DEV)
    flags = torch.zeros(64, dtype=torch.int32, device=DEV)
    p = buf.data_ptr()
    good = dict(inbox=[0, p], peer=[0, p], pflags=[0, flags.data_ptr()])
    bad_cases = [
        dict(good, inbox=[0, 0]),                      # missing inbox for rack 1
        dict(good, inbox=[0, p + 16]),                 # misaligned inbox
        dict(good, peer=[0, p + 4]),                   # misaligned peer inbox
        dict(good, pflags=[0, flags.data_ptr() + 2]),  # misaligned peer flags
    ]
    for case in bad_cases:
        with pytest.raises(PhubError):
            capi.phub_hier_exchange(hub.ctx, 2, 16384, case["inbox"], case["peer"],
                                    flags.data_ptr(), case["pflags"], 1)
    with pytest.raises(PhubError):                      # flags themselves misaligned
        capi.phub_hier_exchange(hub.ctx, 2, 16384, good["inbox"], good["peer"],
                                flags.data_ptr() + 1, good["pflags"], 1)
    assert hub.iteration == 0
    hub.close()
