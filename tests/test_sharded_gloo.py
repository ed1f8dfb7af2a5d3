"""Multi-process (gloo, CPU) tests of the sharded exchange's host logic."""
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

WORKER = os.path.join(ROOT, "tests", "dist", "gloo_exchange_worker.py")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,name,N,cb", [
    (2, "small", 4, 32768), (2, "tiny", 4, 4096), (4, "tiny", 8, 32768), (2, "small", 2, 64),
    (4, "one", 4, 32768),            # one chunk: three owners own nothing
])
def test_gloo_exchange(world, name, N, cb):
    env = dict(os.environ, OMP_NUM_THREADS="1")
    for _attempt in range(3):          # a just-freed port can be taken before torchrun binds it
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
               f"--master-port={_free_port()}", WORKER, name, str(N), str(cb)]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
        if "EADDRINUSE" not in r.stderr:
            break
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count(" ok: ") == world


def test_plan_bytes_and_hosting():
    from paper_1805_07891_b200.sharded import ExchangePlan
    from workloads import manifest
    m = manifest("vgg19")
    E = sum(m)
    for G in (2, 4, 8):
        plans = [ExchangePlan.build(m, 8, 32768, r, G) for r in range(G)]
        assert sorted(w for p in plans for w in p.hosted()) == list(range(8))
        assert all(p.host_of(w) == p.rank for p in plans for w in p.hosted())
        tot_out = sum(p.nvlink_bytes_out() for p in plans)
        tot_in = sum(p.nvlink_bytes_in() for p in plans)
        assert tot_out == tot_in
        # per-GPU bytes out = 32E(G-1)/G^2 + 4E(G-1)/G (+ padding)
        expect = 32 * E * (G - 1) / G ** 2 + 4 * E * (G - 1) / G
        assert abs(max(p.nvlink_bytes_out() for p in plans) / expect - 1) < 2e-3


def test_chain_pieces_and_bytes():
    from paper_1805_07891_b200.sharded import ExchangePlan, chain_nvlink_bytes, chain_pieces
    for Ep, k in ((32, 3), (143667264, 8), (288768, 16), (64, 64), (143667264, 1)):
        p = chain_pieces(Ep, k)
        assert p[0][0] == 0 and p[-1][1] == Ep and len(p) <= k
        assert all(a[1] == b[0] for a, b in zip(p, p[1:]))
        assert all(b % 64 == 0 for b, _ in p)
    # the chain moves fewer NVLink bytes than the owner-sharded exchange at G = 2 only
    from workloads import manifest
    m = manifest("vgg19")
    for G in (2, 4, 8):
        plans = [ExchangePlan.build(m, 8, 32768, r, G) for r in range(G)]
        sharded = max(max(p.nvlink_bytes_out(), p.nvlink_bytes_in()) for p in plans)
        chain = max(max(chain_nvlink_bytes(plans[0].E_padded, G, r)) for r in range(G))
        assert (chain < sharded) == (G == 2)


def test_hier_inbox_slots_and_bytes():
    """Hierarchical exchange host logic: every (epoch parity, source rack)
    slot of an owner's inbox is disjoint and inside the 2 x R x L allocation;
    cross-rack bytes are symmetric over ranks and ~2(G-1)/G model sizes."""
    from paper_1805_07891_b200 import capi
    from paper_1805_07891_b200.sharded import hier_nvlink_bytes, hier_slot
    from workloads import manifest
    m = manifest("vgg19")
    for G in (1, 2, 4, 8):
        Ep, _offs, ranges = capi.phub_plan_ranges(m, 32768, G)
        for o, (b, e) in enumerate(ranges):
            L = e - b
            spans = sorted((hier_slot(sl, q, G, L), hier_slot(sl, q, G, L) + L)
                           for sl in range(2) for q in range(G))
            assert spans[0][0] == 0 and spans[-1][1] == 2 * G * L
            assert all(a[1] == c[0] for a, c in zip(spans, spans[1:]))
        outs = [hier_nvlink_bytes(ranges, Ep, r) for r in range(G)]
        assert sum(o for o, _ in outs) == sum(i for _, i in outs)
        expect = 2 * (G - 1) / G * 4 * Ep
        assert max(max(x) for x in outs) <= expect * 1.001 + 4 * 32768


def test_chain_block_choice():
    from paper_1805_07891_b200.sharded import chain_block_for
    from workloads import manifest
    for name, want in (("resnet50", 8192), ("alexnet", 8192), ("resnet269", 12288),
                       ("vgg19", 12288)):
        b = chain_block_for(sum(manifest(name)))
        assert b == want and b % 2048 == 0


SCHED_WORKER = os.path.join(ROOT, "tests", "dist", "gloo_sched_worker.py")


@pytest.mark.parametrize("world,name,N", [(2, "resnet50", 8), (4, "vgg19", 8), (4, "tiny", 8),
                                          (8, "resnet50", 8)])
def test_gloo_sched_programs(world, name, N):
    """Scheduled exchange host logic across processes: each rank plans only its
    own item program; signals and waits match rank by rank (gloo, CPU)."""
    env = dict(os.environ, OMP_NUM_THREADS="1")
    for _attempt in range(3):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
               f"--master-port={_free_port()}", SCHED_WORKER, name, str(N)]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
        if "EADDRINUSE" not in r.stderr:
            break
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count(" ok: ") == world
