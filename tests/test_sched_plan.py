"""Host logic of the scheduled exchange (phub_sched_plan), on
CPU: the item programs every rank gets for a geometry are checked by
simulation, without any arithmetic of the method:

  * ownership: the Nesterov items of rank o cover exactly [bounds[o],
    bounds[o+1]) and the ranks together cover the padded model once;
  * order: every Nesterov input is the sum of all N workers in worker-id order
    from +0 -- the programs are executed symbolically (each buffer block holds
    the tuple of worker ids summed into it, in order), so a wrong stage, a
    skipped rank, a raw slot read from the wrong source or a final sum sent to
    the wrong owner changes the tuple (reading R3);
  * flags: every waited flag is raised by exactly one item of one rank, and no
    flag index is raised twice;
  * deadlock freedom: executing each rank's program strictly in ticket order
    with ONE worker per rank (the tightest case of the k_sched argument) never
    stalls;
  * raw inbox slots written by different (source rank, worker) never overlap.
"""
import pytest

from paper_1805_07891_b200 import capi

T_RAW, T_CHAIN, T_CRAW, T_CFIN = (capi.PHUB_ITEM_RAW_PUSH, capi.PHUB_ITEM_CHAIN,
                                  capi.PHUB_ITEM_CONSUME_RAW, capi.PHUB_ITEM_CONSUME_FINAL)
NOF = capi.PHUB_NO_FLAG


def geometry(Ep, G, raw_frac, weights=None):
    """Owner bounds (multiples of 8) and raw/chain splits."""
    weights = weights or [1.0] * G
    tot = sum(weights)
    b, acc = [0], 0.0
    for o in range(G - 1):
        acc += weights[o]
        b.append(int(Ep * acc / tot) // 8 * 8)
    b.append(Ep)
    split = [b[o] + int((b[o + 1] - b[o]) * raw_frac[o]) // 8 * 8 for o in range(G)]
    return b, split


def simulate(G, W, bounds, split, block, lag, lanes=False, taper=0):
    """lanes=False: each rank runs its whole program in ticket order on ONE
    worker; lanes=True: as k_sched does, producers (RAW_PUSH, CHAIN) and
    consumers (CONSUME_*) in two independent ticket-ordered lanes, one worker
    each (phub_sched_load's stable partition)."""
    progs, nflags = [], None
    for r in range(G):
        items, nf = capi.phub_sched_plan(G, r, W, bounds, split, block, lag, taper)
        assert nflags in (None, nf)
        nflags = nf
        items = list(items)
        if lanes and any(it.type == T_CHAIN for it in items):   # phub_sched_load's rule
            cons = [it for it in items if it.type in (T_CRAW, T_CFIN)]
            progs.append([it for it in items if it.type not in (T_CRAW, T_CFIN)])
            progs.append(cons)
        else:
            progs.append(items)
            if lanes:
                progs.append([])                # the push plan: one lane in key order
    owner = (lambda i: i // 2) if lanes else (lambda i: i)  # noqa: E731
    flags = [[0] * nflags for _ in range(G)]
    raised = [[0] * nflags for _ in range(G)]
    inbox = [dict() for _ in range(G)]          # (lo, hi) -> tuple of worker ids
    raw = [dict() for _ in range(G)]            # (slot q*W+k, lo, hi) -> worker id
    nag = [[] for _ in range(G)]                # (lo, hi, tuple)
    pc = [0] * len(progs)
    local = lambda r: tuple(range(r * W, (r + 1) * W))  # noqa: E731

    def ready(r, it):
        if it.type == T_CRAW:
            return all(flags[r][it.wait_flag + q] for q in range(G) if q != r)
        return it.wait_flag == NOF or flags[r][it.wait_flag] == 1

    def raise_(dst, f):
        assert raised[dst][f] == 0, f"flag {f} of rank {dst} raised twice"
        raised[dst][f] = 1
        flags[dst][f] = 1

    while any(pc[i] < len(progs[i]) for i in range(len(progs))):
        moved = False
        for i in range(len(progs)):
            if pc[i] >= len(progs[i]):
                continue
            r = owner(i)
            it = progs[i][pc[i]]
            if not ready(r, it):
                continue
            key = (it.lo, it.hi)
            if it.type == T_RAW:
                for k in range(W):
                    slot = (r * W + k, it.lo, it.hi)
                    assert slot not in raw[it.dst], "raw slot written twice"
                    raw[it.dst][slot] = r * W + k
                raise_(it.dst, it.signal_flag)
            elif it.type == T_CHAIN:
                acc = (() if it.wait_flag == NOF else inbox[r].pop(key)) + local(r)
                if it.dst >= 0:
                    inbox[it.dst][key] = acc
                    raise_(it.dst, it.signal_flag)
                else:
                    nag[r].append((it.lo, it.hi, acc))
            elif it.type == T_CRAW:
                acc = ()
                for q in range(G):
                    acc += local(r) if q == r else tuple(raw[r][(q * W + k, it.lo, it.hi)]
                                                         for k in range(W))
                nag[r].append((it.lo, it.hi, acc))
            else:
                nag[r].append((it.lo, it.hi, inbox[r].pop(key)))
            pc[i] += 1
            moved = True
        assert moved, f"deadlock: ranks stuck at {pc} of {[len(p) for p in progs]}"
    return nag, raised


GEOMS = [
    # (Ep, G, W, raw fractions per owner, owner weights, block, lag)
    (65536, 1, 8, [0.5], None, 2048, 0),
    (65536, 2, 4, [0.0, 0.0], [0.0, 1.0], 4096, 0),          # the chain (single owner)
    (65536, 2, 4, [0.3, 0.6], None, 2048, 3),
    (98304, 4, 2, [0.53, 0.0, 0.0, 0.17], [0.298, 0.193, 0.193, 0.316], 2048, 0),  # LP mix
    (98304, 4, 2, [1.0, 0.0, 0.0, 0.0], [1, 2, 2, 3], 4096, 5),                   # simple hybrid
    (131072, 8, 1, [1.0] * 8, None, 2048, 2),                                   # push exchange
    (131072, 8, 1, [0.5] * 8, None, 2048, 0),
    (40000, 3, 3, [0.4, 0.0, 0.2], [0.38, 0.15, 0.47], 2048, 1),               # ragged tail
]


@pytest.mark.parametrize("taper", [0, 3])
@pytest.mark.parametrize("lanes", [False, True])
@pytest.mark.parametrize("Ep,G,W,rf,wts,block,lag", GEOMS)
def test_sched_program_semantics(Ep, G, W, rf, wts, block, lag, lanes, taper):
    bounds, split = geometry(Ep, G, rf, wts)
    nag, raised = simulate(G, W, bounds, split, block, lag, lanes, taper)
    N = G * W
    order = tuple(range(N))
    covered = []
    for r in range(G):
        for lo, hi, acc in nag[r]:
            assert acc == order, f"rank {r} [{lo},{hi}): sum order {acc}"
            assert bounds[r] <= lo < hi <= bounds[r + 1], f"rank {r} optimizes [{lo},{hi})"
            covered.append((lo, hi))
    covered.sort()
    pos = 0
    for lo, hi in covered:
        assert lo == pos, f"gap or overlap at {pos}"
        pos = hi
    assert pos == Ep


def test_every_waited_flag_is_raised_once():
    Ep, G, W = 98304, 4, 2
    bounds, split = geometry(Ep, G, [0.5, 0.0, 0.25, 0.1])
    progs = [capi.phub_sched_plan(G, r, W, bounds, split, 2048, 1)[0] for r in range(G)]
    signals = {}
    for r, prog in enumerate(progs):
        for it in prog:
            if it.dst >= 0:
                k = (it.dst, it.signal_flag)
                assert k not in signals
                signals[k] = r
    for r, prog in enumerate(progs):
        for it in prog:
            if it.type == T_CRAW:
                for q in range(G):
                    if q != r:
                        assert signals[(r, it.wait_flag + q)] == q
            elif it.wait_flag != NOF:
                assert (r, it.wait_flag) in signals


def test_endpoints_match_push_exchange_and_chain():
    """All-RAW parts give the push exchange's items (no chain items); all-CHAIN
    on the last owner gives the chained exchange (no raw items)."""
    Ep = 65536
    b, sp = geometry(Ep, 4, [1.0] * 4)
    for r in range(4):
        items, _ = capi.phub_sched_plan(4, r, 2, b, sp, 2048, 0)
        assert {it.type for it in items} == {T_RAW, T_CRAW}
    b = [0, 0, Ep]
    for r in range(2):
        items, _ = capi.phub_sched_plan(2, r, 4, b, [0, 0], 4096, 0)
        assert {it.type for it in items} == {T_CHAIN}
        assert all((it.dst == -1) == (r == 1) for it in items)


@pytest.mark.parametrize("bad", [
    dict(block=1000), dict(bounds=[8, 100, 200]), dict(split=[0, 300]), dict(bounds=[0, 101, 200]),
    dict(rank=2), dict(W=0),
])
def test_plan_rejects_bad_geometry(bad):
    kw = dict(G=2, rank=0, W=4, bounds=[0, 104, 200], split=[0, 104], block=2048)
    kw.update(bad)
    with pytest.raises(capi.PhubError) as e:
        capi.phub_sched_plan(kw["G"], kw["rank"], kw["W"], kw["bounds"], kw["split"], kw["block"])
    assert capi.STATUS_NAMES[e.value.status] == "PHUB_ERR_INVALID_ARGUMENT"


def test_lp_table_is_balanced():
    """The owner weights / raw fractions sharded.py uses come from the byte
    model of scripts/sched_lp.py: the busiest NVLink port moves at most the
    model's optimum (and never more than the push exchange)."""
    from paper_1805_07891_b200.sharded import SCHED_TABLE, sched_port_bytes
    best = {2: 1.0, 3: 1.7692, 4: 1.7895, 8: 1.75}       # scripts/sched_lp.py optimum
    for G, (wts, rf) in SCHED_TABLE.items():
        W = 8 // G if 8 % G == 0 else 3
        loads = sched_port_bytes(G, W, wts, rf)
        push = sched_port_bytes(G, W, [1.0 / G] * G, [1.0] * G)
        assert max(push) == pytest.approx(1 + (G * W - W - 1) / G)   # closed form, push exchange
        assert max(loads) <= max(push) + 1e-9
        assert max(loads) == pytest.approx(best[G], abs=2e-4)
        assert abs(sum(wts) - 1) < 1e-3 and all(0 <= r <= 1 for r in rf)


def test_taper_cuts_the_ends_finer():
    """taper_blocks: the first and last taper * block elements of every part
    come in blocks of block/4, the middle in whole blocks, covering the part."""
    Ep, block = 196608, 8192                  # 2 x 16384 ends + 20 whole blocks
    b, sp = [0, Ep], [0, 0]                   # one owner, all chain
    items, _ = capi.phub_sched_plan(1, 0, 2, b, sp, block, 0, 2)
    sizes = sorted((it.lo, it.hi - it.lo) for it in items)
    assert sizes[0][0] == 0 and sum(n for _, n in sizes) == Ep
    assert [n for _, n in sizes[:8]] == [2048] * 8              # 2 blocks' worth, 4x finer
    assert [n for _, n in sizes[-8:]] == [2048] * 8
    assert all(n == block for _, n in sizes[8:-8])


@pytest.mark.parametrize("name", ["vgg19", "resnet50", "resnet269", "tiny"])
@pytest.mark.parametrize("G", [2, 4, 8])
def test_geometry_snaps_to_chunk_starts(name, G):
    """sharded.sched_geometry: every owner bound and RAW/CHAIN split is a chunk
    start of the padded layout (each chunk has exactly one owner),
    bounds are monotone from 0 to E_padded, and each owner's share is within
    one chunk of the table's target."""
    from paper_1805_07891_b200.sharded import SCHED_TABLE, sched_geometry
    from workloads import manifest
    sizes = manifest(name)
    wts, rf = SCHED_TABLE[G]
    Ep, bounds, split = sched_geometry(sizes, 32768, G, wts, rf)
    _, offs, _ = capi.phub_plan_ranges(sizes, 32768, 1)
    chunks, n = capi.phub_plan_chunks(sizes, 32768, 1, capi.PHUB_OWNER_CONTIG)
    starts = {int(offs[chunks[i].key_id]) + int(chunks[i].offset) for i in range(n)} | {Ep}
    assert bounds[0] == 0 and bounds[-1] == Ep
    assert all(a <= b for a, b in zip(bounds, bounds[1:]))
    for o in range(G):
        assert bounds[o] in starts and split[o] in starts
        assert bounds[o] <= split[o] <= bounds[o + 1]
    if name != "tiny":                        # 37 chunks: too coarse for the shares
        for o in range(G):
            target = Ep * sum(wts[:o + 1]) / sum(wts)
            assert abs(bounds[o + 1] - target) <= 8192 + 32      # one 32 KB chunk + padding


def test_random_geometries_property():
    """Property check over random plans (hypothesis, bounded): any G in 1..8,
    W in 1..4, owner shares, RAW fractions, block size, lag and taper give
    programs whose symbolic execution sums every element in worker order
    exactly once at its owner, raises every flag once and never stalls --
    with one worker per rank and with the two ticket lanes."""
    hyp = pytest.importorskip("hypothesis")
    st = hyp.strategies

    @hyp.settings(max_examples=60, deadline=None, derandomize=True)
    @hyp.given(G=st.integers(1, 8), W=st.integers(1, 4), data=st.data())
    def check(G, W, data):
        Ep = data.draw(st.integers(1, 24)) * 2048 + data.draw(st.integers(0, 255)) * 8
        wts = [data.draw(st.floats(0.0, 1.0)) + 1e-3 for _ in range(G)]
        rf = [data.draw(st.sampled_from([0.0, 0.25, 0.5, 1.0, data.draw(st.floats(0, 1))]))
              for _ in range(G)]
        block = data.draw(st.sampled_from([2048, 4096, 8192]))
        lag = data.draw(st.integers(0, 8))
        taper = data.draw(st.integers(0, 3))
        lanes = data.draw(st.booleans())
        bounds, split = geometry(Ep, G, rf, wts)
        nag, _ = simulate(G, W, bounds, split, block, lag, lanes, taper)
        order = tuple(range(G * W))
        covered = sorted((lo, hi) for r in range(G) for lo, hi, acc in nag[r]
                         if acc == order and bounds[r] <= lo < hi <= bounds[r + 1])
        assert sum(len(nag[r]) for r in range(G)) == len(covered)
        pos = 0
        for lo, hi in covered:
            assert lo == pos
            pos = hi
        assert pos == Ep

    check()
