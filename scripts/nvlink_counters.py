"""NVLink traffic of the exchange kernels, observed with hardware counters.

One process drives every GPU of the box (G = visible GPUs, 2 or 4): one PHub
context per device wired exactly like sharded.py does across processes
(inboxes, per-block flags, peer replicas -- here plain UVA pointers with peer
access enabled).  Each exchange kernel is launched once per rank with its
real arguments.  Under ncu the launches are serialised, so the device-side
waits are satisfied up front by pre-raising every flag to the epoch: a
launch then moves exactly the bytes of a real round (its data is not a valid
round -- parity is tests/test_gpu_emulated_ranks.py and tests/test_gpu_multi.py).

    ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,... python scripts/nvlink_counters.py vgg19

Prints the analytic NVLink bytes per launch and direction (what bench.py's
roofline_nvlink assumes) as JSON lines, to compare with the counters.
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1805_07891_b200 import PHub, capi  # noqa: E402
from paper_1805_07891_b200.sharded import chain_block_for, hier_slot  # noqa: E402
from workloads import manifest  # noqa: E402


def enable_peer_access(G):
    """cudaDeviceEnablePeerAccess for every ordered pair (primary contexts, shared
    with torch and libphub); refuses to continue if any pair cannot."""
    import ctypes as C
    rt = C.CDLL("/usr/local/cuda/lib64/libcudart.so.12")
    for a in range(G):
        torch.ones(1, device=f"cuda:{a}")          # primary context exists
        for b in range(G):
            if a == b:
                continue
            can = C.c_int()
            assert rt.cudaDeviceCanAccessPeer(C.byref(can), a, b) == 0 and can.value, (a, b)
            assert rt.cudaSetDevice(a) == 0
            e = rt.cudaDeviceEnablePeerAccess(b, 0)
            assert e in (0, 704), f"cudaDeviceEnablePeerAccess({a}->{b}) = {e}"   # 704: enabled
    torch.cuda.synchronize()


def racks(sizes, G, P, worker_order, block):
    hubs = [PHub(sizes, P, device=r, rescale=1.0 / (G * P), num_owners=G, owner_rank=r,
                 owner_policy="contig") for r in range(G)]
    Ep = hubs[0].E_padded
    ranges = [h.owner_range() for h in hubs]
    S = P if worker_order else 1
    grads = [[torch.zeros(Ep, device=f"cuda:{r}") for _ in range(P)] for r in range(G)]
    inbox = [torch.zeros(2 * G * S * max(e - b, 1), device=f"cuda:{r}")
             for r, (b, e) in enumerate(ranges)]
    nblk = [max(1, -(-(e - b) // block)) for b, e in ranges]
    flags = [torch.zeros(n * G, dtype=torch.int32, device=f"cuda:{r}") for r, n in enumerate(nblk)]
    for r, h in enumerate(hubs):
        capi.phub_set_replicas(h.ctx, [hubs[q].weights_ptr() for q in range(G) if q != r])
    return hubs, ranges, grads, inbox, flags, S


def run_racks(sizes, G, P, worker_order, block, epoch=1):
    hubs, ranges, grads, inbox, flags, S = racks(sizes, G, P, worker_order, block)
    par = epoch % 2
    for f in flags:
        f.fill_(epoch)                                   # waits satisfied: launches serialise
    torch.cuda.synchronize()
    for r, h in enumerate(hubs):
        b, e = ranges[r]
        ib, pib, pf = [0] * G, [0] * G, [0] * G
        for o in range(G):
            if o == r:
                continue
            ob, oe = ranges[o]
            ib[o] = inbox[r].data_ptr() + 4 * hier_slot(par, o, G, S * (e - b)) - 4 * b
            pib[o] = inbox[o].data_ptr() + 4 * hier_slot(par, r, G, S * (oe - ob)) - 4 * ob
            pf[o] = flags[o].data_ptr()
        for k in range(P):
            h.push(k, grads[r][k])
        capi.phub_hier_exchange(h.ctx, G, block, ib, pib, flags[r].data_ptr(), pf, epoch,
                                torch.cuda.current_stream(r).cuda_stream,
                                worker_order=worker_order)
        torch.cuda.synchronize(r)
    for r, h in enumerate(hubs):
        b, e = ranges[r]
        L = [oe - ob for ob, oe in ranges]
        if worker_order:
            out = P * sum(4 * L[o] for o in range(G) if o != r) + (G - 1) * 4 * L[r]
            inn = (G - 1) * P * 4 * L[r] + sum(4 * L[o] for o in range(G) if o != r)
        else:
            out = sum(4 * L[o] for o in range(G) if o != r) + (G - 1) * 4 * L[r]
            inn = (G - 1) * 4 * L[r] + sum(4 * L[o] for o in range(G) if o != r)
        print(json.dumps({"kernel": "k_hier", "worker_order": int(worker_order), "G": G,
                          "rank": r, "P": P, "block": block,
                          "analytic_out_bytes": out, "analytic_in_bytes": inn,
                          "timeouts": capi.phub_sync_timeouts(h.ctx)}))
    for h in hubs:
        capi.phub_set_replicas(h.ctx, [])
        h.close()


def run_chain(sizes, N):
    """G = 2 chain: rank 0's k_blocks partial-sum producer -> rank 1's fused consumer."""
    P = N // 2
    prod = PHub(sizes, P, device=0)
    cons = PHub(sizes, P + 1, device=1, rescale=1.0 / N)
    Ep = prod.E_padded
    block = chain_block_for(Ep)
    g0 = [torch.zeros(Ep, device="cuda:0") for _ in range(P)]
    g1 = [torch.zeros(Ep, device="cuda:1") for _ in range(P)]
    inbox = torch.zeros(Ep, device="cuda:1")
    flags = torch.zeros(-(-Ep // block), dtype=torch.int32, device="cuda:1")
    capi.phub_set_replicas(cons.ctx, [prod.weights_ptr()])
    capi.phub_partial_sum(prod.ctx, [g.data_ptr() for g in g0], inbox.data_ptr(), 0, Ep,
                          torch.cuda.current_stream(0).cuda_stream, signal=(flags.data_ptr(), 1),
                          block=block)
    torch.cuda.synchronize(0)
    cons.push(0, inbox)
    for k in range(P):
        cons.push(1 + k, g1[k])
    capi.phub_aggregate_range(cons.ctx, 0, Ep, torch.cuda.current_stream(1).cuda_stream,
                              wait=(flags.data_ptr(), 1), block=block)
    torch.cuda.synchronize(1)
    print(json.dumps({"kernel": "k_blocks producer", "G": 2, "rank": 0,
                      "analytic_out_bytes": 4 * Ep, "analytic_in_bytes": 0}))
    print(json.dumps({"kernel": "k_blocks consumer (fused NAG)", "G": 2, "rank": 1,
                      "analytic_out_bytes": 4 * Ep, "analytic_in_bytes": 0,
                      "timeouts": capi.phub_sync_timeouts(cons.ctx)}))
    capi.phub_set_replicas(cons.ctx, [])
    prod.close()
    cons.close()


def run_p2p(sizes, G, N):
    """Owner-sharded peer-load kernel (P2PShardedPHub): owner r's k_flat loads its
    remote workers' slices over NVLink and stores w' into every peer replica."""
    P = N // G
    hubs = [PHub(sizes, N, device=r, num_owners=G, owner_rank=r, owner_policy="contig")
            for r in range(G)]
    Ep = hubs[0].E_padded
    grads = {w: torch.zeros(Ep, device=f"cuda:{w // P}") for w in range(N)}
    for r, h in enumerate(hubs):
        capi.phub_set_replicas(h.ctx, [hubs[q].weights_ptr() for q in range(G) if q != r])
        for w in range(N):
            h.push(w, grads[w])
        h.aggregate_optimize(stream=torch.cuda.current_stream(r).cuda_stream)
        torch.cuda.synchronize(r)
        b, e = h.owner_range()
        print(json.dumps({"kernel": "k_flat p2p", "G": G, "rank": r,
                          "analytic_out_bytes": (G - 1) * 4 * (e - b),
                          "analytic_in_bytes": (N - P) * 4 * (e - b)}))
    for h in hubs:
        capi.phub_set_replicas(h.ctx, [])
        h.close()


def run_sched(sizes, G, N, block=16384, epoch=1):
    """Scheduled exchange (SchedShardedPHub): one k_sched launch
    per rank with its item program; every flag pre-raised (launches serialise
    under ncu)."""
    from paper_1805_07891_b200.sharded import SCHED_TABLE, sched_geometry, sched_nvlink_bytes
    W = N // G
    wts, rf = SCHED_TABLE.get(G, ([1.0 / G] * G, [1.0] * G))
    Ep, bounds, split = sched_geometry(sizes, 32768, G, wts, rf)
    hubs = [PHub(sizes, W, device=r, rescale=1.0 / N) for r in range(G)]
    grads = [[torch.zeros(Ep, device=f"cuda:{r}") for _ in range(W)] for r in range(G)]
    inbox = [torch.zeros(Ep, device=f"cuda:{r}") for r in range(G)]
    raw = [torch.zeros(G * W * max(split[r] - bounds[r], 8), device=f"cuda:{r}") for r in range(G)]
    flags = []
    for r, h in enumerate(hubs):
        items, nf = capi.phub_sched_plan(G, r, W, bounds, split, block, 0)
        capi.phub_sched_load(h.ctx, G, r, items, nf)
        flags.append(torch.full((max(nf, 1),), epoch, dtype=torch.int32, device=f"cuda:{r}"))
        capi.phub_set_replicas(h.ctx, [hubs[q].weights_ptr() for q in range(G) if q != r])
    torch.cuda.synchronize()
    ptr = lambda ts: [t.data_ptr() for t in ts]  # noqa: E731
    for r, h in enumerate(hubs):
        for k in range(W):
            h.push(k, grads[r][k])
        capi.phub_sched_exchange(h.ctx, ptr(inbox), ptr(raw), ptr(flags), epoch,
                                 torch.cuda.current_stream(r).cuda_stream)
        torch.cuda.synchronize(r)
        out, inn = sched_nvlink_bytes(bounds, split, W, r)
        print(json.dumps({"kernel": "k_sched", "G": G, "rank": r, "W": W, "block": block,
                          "analytic_out_bytes": out, "analytic_in_bytes": inn,
                          "timeouts": capi.phub_sync_timeouts(h.ctx)}))
    for h in hubs:
        capi.phub_set_replicas(h.ctx, [])
        h.close()


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "vgg19"
    sizes = manifest(name)
    G = torch.cuda.device_count()
    enable_peer_access(G)
    if G == 2:
        run_chain(sizes, 8)
    run_racks(sizes, G, 8 // G, True, 12288)              # push exchange (bench default G >= 3)
    run_racks(sizes, G, 8, False, 32768)                  # hierarchical reduction (8 per rack)
    run_p2p(sizes, G, 8)
    run_sched(sizes, G, 8)                                # scheduled exchange (8.6)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "sched":      # the scheduled exchange only
        enable_peer_access(torch.cuda.device_count())
        run_sched(manifest(sys.argv[1]), torch.cuda.device_count(), 8)
    else:
        main()
