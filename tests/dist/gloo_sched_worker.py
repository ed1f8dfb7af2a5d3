"""World-size-N gloo run of the scheduled exchange's host logic on CPU (test
helper for tests/test_sharded_gloo.py).  Every rank derives the geometry
(sharded.sched_geometry) and plans only ITS OWN item program
(phub_sched_plan), as SchedShardedPHub does; the ranks then exchange what they
signal and wait for (all_gather_object) and check, distributed:
  * every rank derived the same owner bounds, splits and flag count;
  * every flag a rank waits on is raised by exactly one item of the rank the
    protocol names (the previous chain stage, the last stage for a final sum,
    rank q for raw slot q), and nothing raises a flag nobody waits on;
  * the per-rank NVLink byte counts balance (sum out == sum in) and the
    busiest port matches the byte model of the owner shares.
"""
import os
import sys

import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_1805_07891_b200 import capi  # noqa: E402
from paper_1805_07891_b200.sharded import (SCHED_TABLE, sched_geometry,  # noqa: E402
                                           sched_nvlink_bytes, sched_port_bytes)
from workloads import manifest  # noqa: E402


def main():
    name, N = sys.argv[1], int(sys.argv[2])
    dist.init_process_group("gloo")
    rank, G = dist.get_rank(), dist.get_world_size()
    W = N // G
    sizes = manifest(name)
    wts, rf = SCHED_TABLE.get(G, ([1.0 / G] * G, [1.0] * G))
    Ep, bounds, split = sched_geometry(sizes, 32768, G, wts, rf)
    items, nf = capi.phub_sched_plan(G, rank, W, bounds, split, 16384, 0)
    sig = sorted((it.dst, it.signal_flag, it.type) for it in items if it.dst >= 0)
    waits = []
    for it in items:
        if it.type == capi.PHUB_ITEM_CONSUME_RAW:
            waits += [(it.wait_flag + q, q) for q in range(G) if q != rank]
        elif it.wait_flag != capi.PHUB_NO_FLAG:
            src = rank - 1 if it.type == capi.PHUB_ITEM_CHAIN else G - 1
            waits.append((it.wait_flag, src))
    mine = (rank, bounds, split, nf, sig, waits, sched_nvlink_bytes(bounds, split, W, rank))
    allr = [None] * G
    dist.all_gather_object(allr, mine)
    allr.sort(key=lambda x: x[0])
    assert all(x[1] == bounds and x[2] == split and x[3] == nf for x in allr), "geometry differs"
    raised = {}
    for q, *_rest in allr:
        for dst, f, _t in allr[q][4]:
            assert (dst, f) not in raised, f"flag {f} of rank {dst} raised twice"
            raised[(dst, f)] = q
    waited = set()
    for f, src in waits:
        assert raised.get((rank, f)) == src, f"rank {rank} waits on flag {f} from {src}"
        waited.add((rank, f))
    mine_raised = {k for k in raised if k[0] == rank}
    assert mine_raised == waited, f"rank {rank}: raised but never waited {mine_raised - waited}"
    outs = [x[6][0] for x in allr]
    ins = [x[6][1] for x in allr]
    assert sum(outs) == sum(ins)
    model = sched_port_bytes(G, W, [(bounds[o + 1] - bounds[o]) / Ep for o in range(G)],
                             [(split[o] - bounds[o]) / max(bounds[o + 1] - bounds[o], 1)
                              for o in range(G)])
    busiest = max(max(o, i) for o, i in zip(outs, ins)) / (4 * Ep)
    assert abs(busiest - max(model)) < 1e-6, (busiest, model)
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank}/{G} ok: {len(items)} items, busiest port {busiest:.4f} model sizes")


if __name__ == "__main__":
    main()
