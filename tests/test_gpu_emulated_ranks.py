"""The multi-GPU exchange kernels with R ranks emulated on ONE B200 (-m gpu;
VERDICT r1 "next" #2): R contexts on one device, each owning a CONTIG range,
each launched on its own stream so the ranks' kernels run CONCURRENTLY and
really exchange through the flag protocols (grids capped with PHUB_OPT_GRID so
every rank's CTAs are co-resident).  Local device buffers stand in for the
peer-mapped inboxes, flags and replicas -- the same addresses a rank would get
from phub_ipc_open, with the same per-epoch slot arithmetic as
sharded.hier_slot.

Covered (the defaults of sharded.py at G >= 2):
  * k_hier worker_order = 1: the owner-sharded push exchange of ONE job
    (PushShardedPHub), R = 2, 4 -- bit-exact vs oracle.round_ over all R*P
    workers in global worker order;
  * k_hier worker_order = 0: hierarchical reduction (HierPHub), R = 2, 4 --
    bit-exact vs oracle.hier_round, and DIFFERENT from the flat order at R = 2
    (rack grouping is visible with full-mantissa inputs);
  * the block-streamed chain (ChainShardedPHub, sync="blocks"): producer and
    consumer kernels on different streams, the consumer launched FIRST so it
    really waits on the producer's per-block flags; and the per-piece "flags"
    chain (k_prefix -> k_flat with stage flags);
  * an expired wait: one rank of a push exchange never launched -> the other
    rank's next call fails with PHUB_ERR_SYNC_TIMEOUT;
  * k_sched (SchedShardedPHub, the multi-GPU default since round 2): the item
    programs of the chain plan (R = 2), the LP mixes (R = 3, 4), a hybrid and
    the push plan (R = 8), bit-exact vs the worker-order oracle, and its
    missing-rank timeout.
Every case asserts phub_sync_timeouts == 0 (except the forced one).
"""
import numpy as np
import pytest

import oracle
from workloads import grad_stream, manifest
from workloads.generate import fullmant_np

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

f32 = np.float32
DEV = "cuda:0"


def bits(a):
    return np.asarray(a, dtype=f32).view(np.uint32)


def assert_bits_equal(got, ref, what):
    got, ref = np.asarray(got, f32), np.asarray(ref, f32)
    bad = np.flatnonzero(bits(got) != bits(ref))
    assert bad.size == 0, f"{what}: {bad.size} of {ref.size} elements differ, first {bad[:5]}"


def hier_slot(slot, src, racks, owned):
    return (slot * racks + src) * owned      # == sharded.hier_slot (kept independent here)


class EmulatedRacks:
    """R rack contexts on one GPU wired like HierPHub / PushShardedPHub."""

    def __init__(self, sizes, R, P, worker_order, block, grid, seed, lr=0.1, mu=0.9):
        from paper_1805_07891_b200 import PHub, capi
        self.capi = capi
        self.R, self.P, self.wo, self.block = R, P, worker_order, block
        self.hubs = [PHub(sizes, P, device=0, lr=lr, momentum=mu, rescale=1.0 / (R * P),
                          num_owners=R, owner_rank=r, owner_policy="contig", keep_aggregate=True)
                     for r in range(R)]
        h0 = self.hubs[0]
        self.E, self.Ep = h0.E, h0.E_padded
        self.ranges = [h.owner_range() for h in self.hubs]
        S = P if worker_order else 1
        self.S = S
        self.inbox = [torch.zeros(2 * R * S * max(e - b, 1), device=DEV) for b, e in self.ranges]
        # block flags sized by the largest owner range on every rank, + the 2R
        # round-barrier flags (phub_hier.device_barrier)
        J = max(max(1, -(-(e - b) // block)) for b, e in self.ranges)
        self.flags = [torch.zeros(J * R + 2 * R, dtype=torch.int32, device=DEV) for _ in range(R)]
        self.streams = [torch.cuda.Stream() for _ in range(R)]
        for r, h in enumerate(self.hubs):
            h.set_option(capi.PHUB_OPT_GRID, grid)
            capi.phub_set_replicas(h.ctx, [self.hubs[q].weights_ptr() for q in range(R) if q != r])
        self.epoch = 0
        self.seed = seed
        idx = torch.as_tensor(h0.padded_index(), device=DEV)
        from workloads.generate import fullmant_torch
        # rack q's local worker k is global worker q*P + k
        self.grads = []
        for q in range(R):
            rack = []
            for k in range(P):
                b = torch.full((self.Ep,), float("nan"), device=DEV)
                b[idx] = fullmant_torch(grad_stream(q * P + k) + 37 * seed, 0, self.E, DEV)
                rack.append(b)
            self.grads.append(rack)

    def host_grads(self):
        return [[fullmant_np(grad_stream(q * self.P + k) + 37 * self.seed, 0, self.E)
                 for k in range(self.P)] for q in range(self.R)]

    def load_state(self, w, v):
        for h in self.hubs:
            h.load_state(w, v)

    def pointers(self, r, par):
        R, S = self.R, self.S
        b, e = self.ranges[r]
        inbox, peer_inbox, peer_flags = [0] * R, [0] * R, [0] * R
        for o in range(R):
            if o == r:
                continue
            ob, oe = self.ranges[o]
            inbox[o] = self.inbox[r].data_ptr() + 4 * hier_slot(par, o, R, S * (e - b)) - 4 * b
            peer_inbox[o] = self.inbox[o].data_ptr() + 4 * hier_slot(par, r, R, S * (oe - ob)) \
                - 4 * ob
            peer_flags[o] = self.flags[o].data_ptr()
        return inbox, peer_inbox, peer_flags

    def round(self, ranks=None, order=None, device_barrier=False):
        self.epoch += 1
        par = self.epoch % 2
        if not device_barrier:
            torch.cuda.synchronize()                 # start barrier (replicas free)
        for r in (order or range(self.R)):
            if ranks is not None and r not in ranks:
                continue
            h = self.hubs[r]
            for k in range(self.P):
                h.push(k, self.grads[r][k])
            inbox, peer_inbox, peer_flags = self.pointers(r, par)
            self.capi.phub_hier_exchange(h.ctx, self.R, self.block, inbox, peer_inbox,
                                         self.flags[r].data_ptr(), peer_flags, self.epoch,
                                         self.streams[r].cuda_stream, worker_order=self.wo,
                                         device_barrier=device_barrier)
        if not device_barrier:
            torch.cuda.synchronize()                 # end barrier (replicas complete)

    def close(self):
        for h in self.hubs:
            h.close()


SMALL = [3, 3, 9408, 64, 64, 4096, 20000, 1000, 262144, 7]


@pytest.mark.parametrize("R,P,name,block,rounds", [
    (2, 4, "small", 2048, 2), (4, 2, "small", 2048, 2), (2, 4, "resnet50", 12288, 2),
    (4, 2, "resnet50", 12288, 2), (4, 1, "tiny", 2048, 3), (8, 1, "resnet50", 12288, 2)])
def test_push_exchange_emulated(R, P, name, block, rounds):
    """k_hier worker_order=1 == PushShardedPHub's round: bit-exact vs the
    worker-order oracle over all R*P workers; every rank holds the full w'."""
    sizes = SMALL if name == "small" else manifest(name)
    em = EmulatedRacks(sizes, R, P, True, block, grid=max(1, 360 // R), seed=60 + R)
    w, v = fullmant_np(1 + 37 * 60, 0, em.E), fullmant_np(2 + 37 * 60, 0, em.E)
    em.load_state(w, v)
    flat = [g for rack in em.host_grads() for g in rack]
    for _ in range(rounds):
        em.round(order=list(reversed(range(R))))       # a launch order unlike worker order
        w, v, s = oracle.round_(sizes, flat, w, v, 0.1, 0.9)
    for r, h in enumerate(em.hubs):
        assert em.capi.phub_sync_timeouts(h.ctx) == 0
        gw, gv, gs = h.read_state()
        assert_bits_equal(gw, w, f"rank {r} replica w'")
        own = _owned_mask(h, sizes)
        assert_bits_equal(gv[own], v[own], f"rank {r} owned v'")
        assert_bits_equal(gs[own], s[own], f"rank {r} owned s")
    em.close()


def _owned_mask(h, sizes):
    tab = h.chunk_table()
    starts = np.concatenate([[0], np.cumsum(sizes)])
    m = np.zeros(int(sum(sizes)), bool)
    for k, off, ln, own in zip(tab["key_id"], tab["offset"], tab["length"], tab["owner"]):
        if own == h.owner_rank:
            a = int(starts[k] + off)
            m[a:a + int(ln)] = True
    return m


@pytest.mark.parametrize("R,P,name,block", [
    (2, 4, "small", 2048), (4, 2, "small", 2048), (2, 8, "resnet50", 32768),
    (4, 3, "resnet50", 16384), (8, 2, "small", 2048)])
def test_hierarchical_exchange_emulated(R, P, name, block):
    """k_hier worker_order=0 == HierPHub's round: bit-exact vs
    oracle.hier_round (rack-order sum of rack aggregates, reading R17), and
    -- with full-mantissa inputs -- NOT equal to the flat worker-order sum."""
    sizes = SMALL if name == "small" else manifest(name)
    em = EmulatedRacks(sizes, R, P, False, block, grid=max(1, 360 // R), seed=70 + R)
    w0, v0 = fullmant_np(1 + 37 * 70, 0, em.E), fullmant_np(2 + 37 * 70, 0, em.E)
    em.load_state(w0, v0)
    rg = em.host_grads()
    em.round()
    w, v, s = oracle.hier_round(sizes, rg, w0, v0, 0.1, 0.9)
    _, _, flat_s = oracle.round_(sizes, [g for rack in rg for g in rack], w0, v0, 0.1, 0.9)
    assert np.mean(bits(s) != bits(flat_s)) > 0.05          # rack order is visible
    for r, h in enumerate(em.hubs):
        assert em.capi.phub_sync_timeouts(h.ctx) == 0
        gw, gv, gs = h.read_state()
        assert_bits_equal(gw, w, f"rank {r} replica w'")
        own = _owned_mask(h, sizes)
        assert_bits_equal(gs[own], s[own], f"rank {r} owned s (hierarchical)")
        assert_bits_equal(gv[own], v[own], f"rank {r} owned v'")
    em.close()


def test_push_exchange_missing_rank_times_out_loudly():
    """Rank 1 never launches: rank 0's consume waits expire (~2 s), its blocks
    are skipped, and its context is sticky-failed -- the next call and every
    synchronizing call report PHUB_ERR_SYNC_TIMEOUT instead of a stale w'."""
    from paper_1805_07891_b200 import PhubError
    em = EmulatedRacks(manifest("tiny"), 2, 2, True, 2048, grid=64, seed=80)
    em.round(ranks=[0])
    h = em.hubs[0]
    assert em.capi.phub_sync_timeouts(h.ctx) >= 1
    for fn in (lambda: h.push(0, em.grads[0][0]), h.read_state, h.synchronize):
        with pytest.raises(PhubError) as e:
            fn()
        assert em.capi.STATUS_NAMES[e.value.status] == "PHUB_ERR_SYNC_TIMEOUT"
    assert em.capi.phub_check(em.hubs[1].ctx) == 0            # the other rank never waited
    em.close()


@pytest.mark.parametrize("block,name", [(2048, "small"), (12288, "resnet50"), (8192, "tiny")])
def test_block_chain_concurrent_streams(block, name):
    """ChainShardedPHub at G = 2 on one GPU: rank 0's k_blocks producer stores
    its partial block by block into rank 1's inbox and raises per-block flags;
    rank 1's fused k_blocks consumer -- launched FIRST on its own stream --
    waits on each flag, finishes the worker-order sum, runs Nesterov and stores
    w' into rank 0's replica.  Bit-exact vs the 2P-worker oracle round."""
    from paper_1805_07891_b200 import PHub, capi
    sizes = SMALL if name == "small" else manifest(name)
    P = 4
    prod = PHub(sizes, P, device=0)
    cons = PHub(sizes, P + 1, device=0, rescale=1.0 / (2 * P), keep_aggregate=True)
    E, Ep = prod.E, prod.E_padded
    w0, v0 = fullmant_np(1 + 37 * 90, 0, E), fullmant_np(2 + 37 * 90, 0, E)
    cons.load_state(w0, v0)
    from workloads.generate import fullmant_torch
    idx = torch.as_tensor(prod.padded_index(), device=DEV)
    gd = []
    for k in range(2 * P):
        b = torch.zeros(Ep, device=DEV)          # finite padding: the partial sum reads it
        b[idx] = fullmant_torch(grad_stream(k) + 37 * 90, 0, E, DEV)
        gd.append(b)
    inbox = torch.zeros(Ep, device=DEV)
    flags = torch.zeros(-(-Ep // block), dtype=torch.int32, device=DEV)
    capi.phub_set_replicas(cons.ctx, [prod.weights_ptr()])
    for h in (prod, cons):
        h.set_option(capi.PHUB_OPT_GRID, 148)
    s_prod, s_cons = torch.cuda.Stream(), torch.cuda.Stream()
    w, v = w0, v0
    hg = [fullmant_np(grad_stream(k) + 37 * 90, 0, E) for k in range(2 * P)]
    for ep in (1, 2):
        cons.push(0, inbox)
        for k in range(P):
            cons.push(1 + k, gd[P + k])
        torch.cuda.synchronize()
        capi.phub_aggregate_range(cons.ctx, 0, Ep, s_cons.cuda_stream, wait=(flags.data_ptr(), ep),
                                  block=block)
        capi.phub_partial_sum(prod.ctx, [g.data_ptr() for g in gd[:P]], inbox.data_ptr(), 0, Ep,
                              s_prod.cuda_stream, signal=(flags.data_ptr(), ep), block=block)
        torch.cuda.synchronize()
        w, v, s = oracle.round_(sizes, hg, w, v, 0.1, 0.9)
    assert capi.phub_sync_timeouts(cons.ctx) == 0 and capi.phub_sync_timeouts(prod.ctx) == 0
    gw, gv, gs = cons.read_state()
    assert_bits_equal(gs, s, "chain aggregate")
    assert_bits_equal(gw, w, "chain w'")
    assert_bits_equal(gv, v, "chain v'")
    pw, _, _ = prod.read_state()
    assert_bits_equal(pw, w, "rank 0 replica (stored by rank 1 over 'NVLink')")
    prod.close()
    cons.close()


def test_piece_flags_chain_concurrent_streams():
    """ChainShardedPHub sync='flags' on one GPU: per-piece k_prefix launches
    raise one flag each; the consumer's per-piece k_flat launches (enqueued
    first, on another stream) wait on them.  Bit-exact vs the oracle."""
    from paper_1805_07891_b200 import PHub, capi
    from paper_1805_07891_b200.sharded import chain_pieces
    sizes = manifest("resnet50")
    P = 3
    prod = PHub(sizes, P, device=0)
    cons = PHub(sizes, P + 1, device=0, rescale=1.0 / (2 * P))
    E, Ep = prod.E, prod.E_padded
    w0, v0 = fullmant_np(1 + 37 * 91, 0, E), fullmant_np(2 + 37 * 91, 0, E)
    cons.load_state(w0, v0)
    from workloads.generate import fullmant_torch
    idx = torch.as_tensor(prod.padded_index(), device=DEV)
    gd = []
    for k in range(2 * P):
        b = torch.zeros(Ep, device=DEV)
        b[idx] = fullmant_torch(grad_stream(k) + 37 * 91, 0, E, DEV)
        gd.append(b)
    inbox = torch.zeros(Ep, device=DEV)
    pieces = chain_pieces(Ep, 6)
    flags = torch.zeros(len(pieces), dtype=torch.int32, device=DEV)
    for h in (prod, cons):
        h.set_option(capi.PHUB_OPT_GRID, 148)
    s_prod, s_cons = torch.cuda.Stream(), torch.cuda.Stream()
    cons.push(0, inbox)
    for k in range(P):
        cons.push(1 + k, gd[P + k])
    torch.cuda.synchronize()         # the zero-fills above ran on torch's stream, not s_*
    for p, (b, e) in enumerate(pieces):
        capi.phub_aggregate_range(cons.ctx, b, e, s_cons.cuda_stream,
                                  wait=(flags.data_ptr() + 4 * p, 1))
    for p, (b, e) in enumerate(pieces):
        capi.phub_partial_sum(prod.ctx, [g.data_ptr() for g in gd[:P]], inbox.data_ptr(), b, e,
                              s_prod.cuda_stream, signal=(flags.data_ptr() + 4 * p, 1))
    torch.cuda.synchronize()
    assert capi.phub_sync_timeouts(cons.ctx) == 0
    hg = [fullmant_np(grad_stream(k) + 37 * 91, 0, E) for k in range(2 * P)]
    w, v, _ = oracle.round_(sizes, hg, w0, v0, 0.1, 0.9)
    gw, gv, _ = cons.read_state()
    assert_bits_equal(gw, w, "piece-chain w'")
    assert_bits_equal(gv, v, "piece-chain v'")
    prod.close()
    cons.close()


# ---------------------------------------------- scheduled exchange (8.6)
class EmulatedSched:
    """R rank contexts of SchedShardedPHub on one GPU: each rank's item program
    (phub_sched_plan) loaded into its own context, launched on its own stream;
    local buffers stand in for the peer-mapped inboxes, raw inboxes, flags and
    replicas."""

    def __init__(self, sizes, R, W, weights, raw_frac, block, lag, grid, seed, cb=32768, taper=0):
        from paper_1805_07891_b200 import PHub, capi
        from paper_1805_07891_b200.sharded import sched_geometry
        self.capi, self.R, self.W, self.seed = capi, R, W, seed
        self.Ep, self.bounds, self.split = sched_geometry(sizes, cb, R, weights, raw_frac)
        self.hubs = [PHub(sizes, W, chunk_size_bytes=cb, device=0, rescale=1.0 / (R * W),
                          keep_aggregate=True) for _ in range(R)]
        h0 = self.hubs[0]
        self.E = h0.E
        self.nflags = None
        for r, h in enumerate(self.hubs):
            items, nf = capi.phub_sched_plan(R, r, W, self.bounds, self.split, block, lag, taper)
            capi.phub_sched_load(h.ctx, R, r, items, nf)
            self.nflags = nf
            h.set_option(capi.PHUB_OPT_GRID, grid)
            capi.phub_set_replicas(h.ctx, [self.hubs[q].weights_ptr() for q in range(R) if q != r])
        self.inbox = [torch.zeros(self.Ep, device=DEV) for _ in range(R)]
        self.raw = [torch.zeros(R * W * max(self.split[r] - self.bounds[r], 8), device=DEV)
                    for r in range(R)]
        self.flags = [torch.zeros(max(self.nflags, 1), dtype=torch.int32, device=DEV)
                      for _ in range(R)]
        self.streams = [torch.cuda.Stream() for _ in range(R)]
        self.epoch = 0
        idx = torch.as_tensor(h0.padded_index(), device=DEV)
        self.pidx = h0.padded_index()
        from workloads.generate import fullmant_torch
        self.grads = []
        for q in range(R):
            rank = []
            for k in range(W):
                b = torch.full((self.Ep,), float("nan"), device=DEV)
                b[idx] = fullmant_torch(grad_stream(q * W + k) + 37 * seed, 0, self.E, DEV)
                rank.append(b)
            self.grads.append(rank)

    def host_grads(self):
        return [fullmant_np(grad_stream(w) + 37 * self.seed, 0, self.E)
                for w in range(self.R * self.W)]

    def owned_mask(self, r):
        return (self.pidx >= self.bounds[r]) & (self.pidx < self.bounds[r + 1])

    def round(self, order=None, device_barrier=False):
        """device_barrier=False: host synchronizes around the round (the caller's
        barriers); True: no host synchronization at all -- the launches' in-kernel
        round barriers alone must order consecutive rounds on the ranks' streams."""
        self.epoch += 1
        if not device_barrier:
            torch.cuda.synchronize()                 # start barrier
        ptr = lambda ts: [t.data_ptr() for t in ts]  # noqa: E731
        for r in (order or range(self.R)):
            h = self.hubs[r]
            for k in range(self.W):
                h.push(k, self.grads[r][k])
            self.capi.phub_sched_exchange(h.ctx, ptr(self.inbox), ptr(self.raw), ptr(self.flags),
                                          self.epoch, self.streams[r].cuda_stream,
                                          device_barrier=device_barrier)
        if not device_barrier:
            torch.cuda.synchronize()                 # end barrier

    def close(self):
        for h in self.hubs:
            h.close()


SCHED_CASES = [
    # R, W, weights, raw fractions, manifest, block, lag, rounds[, taper]
    (2, 4, [0.0, 1.0], [0.0, 0.0], "resnet50", 16384, 0, 2),                  # = the chain
    (2, 4, [0.45, 0.55], [0.5, 0.3], "small", 2048, 1, 2),
    (4, 2, [0.2982, 0.193, 0.193, 0.3158], [0.5294, 0.0, 0.0, 0.1667], "resnet50", 16384, 0, 2),
    (4, 2, [0.2982, 0.193, 0.193, 0.3158], [0.5294, 0.0, 0.0, 0.1667], "small", 2048, 4, 3),
    (4, 2, [0.125, 0.25, 0.25, 0.375], [1.0, 0.0, 0.0, 0.0], "tiny", 2048, 2, 2),
    (8, 1, [0.125] * 8, [1.0] * 8, "resnet50", 16384, 0, 2),                  # = push exchange
    (3, 3, [0.3846, 0.1538, 0.4616], [0.4, 0.0, 0.1667], "small", 2048, 0, 2),  # N = 9
    (4, 2, [0.2982, 0.193, 0.193, 0.3158], [0.5294, 0.0, 0.0, 0.1667], "resnet50", 12288, 64, 2, 4),
]


@pytest.mark.parametrize("case", SCHED_CASES)
def test_sched_exchange_emulated(case):
    """k_sched == SchedShardedPHub's round: bit-exact vs the worker-order oracle
    over all R*W workers on every replica; v' and s bit-exact on each rank's
    Nesterov range."""
    R, W, wts, rf, name, block, lag, rounds = case[:8]
    taper = case[8] if len(case) > 8 else 0
    sizes = SMALL if name == "small" else manifest(name)
    em = EmulatedSched(sizes, R, W, wts, rf, block, lag, grid=max(1, 360 // R), seed=100 + R,
                       taper=taper)
    w, v = fullmant_np(1 + 37 * 100, 0, em.E), fullmant_np(2 + 37 * 100, 0, em.E)
    for h in em.hubs:
        h.load_state(w, v)
    flat = em.host_grads()
    for _ in range(rounds):
        em.round(order=list(reversed(range(R))))
        w, v, s = oracle.round_(sizes, flat, w, v, 0.1, 0.9)
    for r, h in enumerate(em.hubs):
        assert em.capi.phub_sync_timeouts(h.ctx) == 0
        gw, gv, gs = h.read_state()
        assert_bits_equal(gw, w, f"rank {r} replica w'")
        own = em.owned_mask(r)
        assert_bits_equal(gv[own], v[own], f"rank {r} owned v'")
        assert_bits_equal(gs[own], s[own], f"rank {r} owned s")
    em.close()


def test_sched_exchange_missing_rank_times_out_loudly():
    """Rank 1 never launches: rank 0's chain/consume waits expire, the context
    is sticky-failed and the next call reports PHUB_ERR_SYNC_TIMEOUT."""
    from paper_1805_07891_b200 import PhubError
    em = EmulatedSched(manifest("tiny"), 2, 2, [0.5, 0.5], [0.5, 0.5], 2048, 0, grid=64, seed=81)
    em.epoch += 1
    h = em.hubs[0]
    for k in range(2):
        h.push(k, em.grads[0][k])
    ptr = lambda ts: [t.data_ptr() for t in ts]  # noqa: E731
    em.capi.phub_sched_exchange(h.ctx, ptr(em.inbox), ptr(em.raw), ptr(em.flags), em.epoch,
                                em.streams[0].cuda_stream)
    torch.cuda.synchronize()
    assert em.capi.phub_sync_timeouts(h.ctx) >= 1
    with pytest.raises(PhubError) as e:
        h.read_state()
    assert em.capi.STATUS_NAMES[e.value.status] == "PHUB_ERR_SYNC_TIMEOUT"
    em.close()


def test_sched_g8_bench_plan_full_vgg19_emulated():
    """The G = 8 launch configuration bench.py would time on an 8-GPU box --
    SCHED_TABLE[8] (the push plan, one ticket lane), 12K-element blocks, lag
    64, taper 8, one worker per rank -- at BASELINE.json's full VGG-19 size,
    eight ranks emulated on one GPU: every replica bit-exact vs the oracle
    round, every owner's v' and s too (no 8-GPU runner was available)."""
    from paper_1805_07891_b200.sharded import SCHED_TABLE
    wts, rf = SCHED_TABLE[8]
    sizes = manifest("vgg19")
    em = EmulatedSched(sizes, 8, 1, wts, rf, 12288, 64, grid=45, seed=120, taper=8)
    w, v = fullmant_np(1 + 37 * 120, 0, em.E), fullmant_np(2 + 37 * 120, 0, em.E)
    for h in em.hubs:
        h.load_state(w, v)
    em.round(order=list(reversed(range(8))))
    w, v, s = oracle.round_(sizes, em.host_grads(), w, v, 0.1, 0.9)
    for r, h in enumerate(em.hubs):
        assert em.capi.phub_sync_timeouts(h.ctx) == 0
        gw, gv, gs = h.read_state()
        assert_bits_equal(gw, w, f"rank {r} replica w'")
        own = em.owned_mask(r)
        assert_bits_equal(gv[own], v[own], f"rank {r} owned v'")
        assert_bits_equal(gs[own], s[own], f"rank {r} owned s")
    em.close()


@pytest.mark.parametrize("R,W,wts,rf,name,block,lag,taper", [
    (2, 4, [0.0, 1.0], [0.0, 0.0], "resnet50", 16384, 0, 0),
    (4, 2, [0.2982, 0.193, 0.193, 0.3158], [0.5294, 0.0, 0.0, 0.1667], "resnet50", 12288, 64, 8),
    (8, 1, [0.125] * 8, [1.0] * 8, "small", 2048, 0, 0),
])
def test_sched_device_barrier_back_to_back_rounds(R, W, wts, rf, name, block, lag, taper):
    """phub_sched.device_barrier: four rounds enqueued on the ranks' own streams
    with NO host synchronization in between -- a rank may start round k+1 while
    its peers still run round k; the in-kernel start flags keep its w' stores out
    of replicas not yet released, the end flags keep inboxes from being
    overwritten early.  Bit-exact vs four oracle rounds."""
    sizes = SMALL if name == "small" else manifest(name)
    em = EmulatedSched(sizes, R, W, wts, rf, block, lag, grid=max(2, 360 // R), seed=130 + R,
                       taper=taper)
    w, v = fullmant_np(1 + 37 * 130, 0, em.E), fullmant_np(2 + 37 * 130, 0, em.E)
    for h in em.hubs:
        h.load_state(w, v)
    torch.cuda.synchronize()
    flat = em.host_grads()
    for i in range(4):
        em.round(order=list(range(R)) if i % 2 else list(reversed(range(R))), device_barrier=True)
        w, v, s = oracle.round_(sizes, flat, w, v, 0.1, 0.9)
    torch.cuda.synchronize()
    for r, h in enumerate(em.hubs):
        assert em.capi.phub_sync_timeouts(h.ctx) == 0
        gw, gv, gs = h.read_state()
        assert_bits_equal(gw, w, f"rank {r} replica w'")
        own = em.owned_mask(r)
        assert_bits_equal(gv[own], v[own], f"rank {r} owned v'")
        assert_bits_equal(gs[own], s[own], f"rank {r} owned s")
    em.close()


@pytest.mark.parametrize("R,P,wo,name,block", [
    (2, 4, True, "resnet50", 12288), (4, 2, True, "small", 2048),
    (2, 8, False, "resnet50", 32768), (4, 3, False, "small", 2048)])
def test_hier_device_barrier_back_to_back_rounds(R, P, wo, name, block):
    """phub_hier.device_barrier (push exchange wo = 1, hierarchical wo = 0):
    three rounds on the ranks' own streams with NO host synchronization in
    between, ordered only by the in-kernel start / done flags.  Bit-exact vs
    the oracle (flat worker order, or rack order)."""
    sizes = SMALL if name == "small" else manifest(name)
    em = EmulatedRacks(sizes, R, P, wo, block, grid=max(2, 360 // R), seed=140 + R)
    w, v = fullmant_np(1 + 37 * 140, 0, em.E), fullmant_np(2 + 37 * 140, 0, em.E)
    em.load_state(w, v)
    torch.cuda.synchronize()
    rg = em.host_grads()
    for i in range(3):
        em.round(order=list(range(R)) if i % 2 else list(reversed(range(R))), device_barrier=True)
        if wo:
            w, v, s = oracle.round_(sizes, [g for rack in rg for g in rack], w, v, 0.1, 0.9)
        else:
            w, v, s = oracle.hier_round(sizes, rg, w, v, 0.1, 0.9)
    torch.cuda.synchronize()
    for r, h in enumerate(em.hubs):
        assert em.capi.phub_sync_timeouts(h.ctx) == 0
        gw, gv, gs = h.read_state()
        assert_bits_equal(gw, w, f"rank {r} replica w'")
        own = _owned_mask(h, sizes)
        assert_bits_equal(gv[own], v[own], f"rank {r} owned v'")
        assert_bits_equal(gs[own], s[own], f"rank {r} owned s")
    em.close()
