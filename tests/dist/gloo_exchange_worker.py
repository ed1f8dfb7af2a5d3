"""World-size-N gloo run of the sharded exchange schedule on CPU (test helper).

Launched by tests/test_sharded_gloo.py through torch.distributed.run.  The
owner's compute is stood in for by the CPU oracle (this is test code: the
product path never computes on the CPU); what is under test is the host logic
of paper_1805_07891_b200.sharded -- the plan, the push schedule (every owner
receives exactly its workers' slices, in worker order) and the all-gather-v
pull (every replica ends up complete).
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1805_07891_b200 import capi  # noqa: E402
from paper_1805_07891_b200.sharded import ExchangePlan, push_exchange, pull_exchange  # noqa: E402
from workloads import grad_stream, manifest, values_np  # noqa: E402


def main():
    name, N, cb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    special = {"small": [3, 3, 9408, 64, 64, 4096, 20000, 7], "one": [5]}
    sizes = special[name] if name in special else manifest(name)
    E = sum(sizes)
    plan = ExchangePlan.build(sizes, N, cb, rank, world)
    Ep, offs, ranges = capi.phub_plan_ranges(sizes, cb, world)
    pidx = np.concatenate([offs[k] + np.arange(n) for k, n in enumerate(sizes)])
    real_of = np.full(Ep, -1, np.int64)
    real_of[pidx] = np.arange(E)

    hg = [values_np(grad_stream(w), 0, E, 25) for w in range(N)]
    w0, v0 = values_np(1, 0, E, 20), values_np(2, 0, E, 25)
    grads = {}
    for w in plan.hosted():
        t = torch.full((Ep,), float("nan"))
        t[torch.as_tensor(pidx)] = torch.as_tensor(hg[w])
        grads[w] = t
    b, e = plan.owned()
    recv = {w: torch.empty(e - b) for w in range(N) if plan.host_of(w) != rank}
    push_exchange(plan, grads, recv)

    # every owner now holds its workers' slices of [b, e): check them
    sel = real_of[b:e]
    real = sel >= 0
    slices = []
    for w in range(N):
        s = (grads[w][b:e] if plan.host_of(w) == rank else recv[w]).numpy()
        assert np.array_equal(s[real].view(np.uint32), hg[w][sel[real]].view(np.uint32)), \
            f"rank {rank}: worker {w} slice wrong"
        slices.append(s[real])
    # owner compute stand-in (test only): the oracle on the owned real elements
    nw, _, _ = oracle.elems(np.stack(slices), w0[sel[real]], v0[sel[real]], 0.1, 0.9)
    replica = torch.full((Ep,), float("nan"))
    own = torch.as_tensor(np.arange(b, e)[real])
    replica[own] = torch.as_tensor(nw)
    pull_exchange(plan, replica)

    ref_w, _, _ = oracle.round_(sizes, hg, w0, v0, 0.1, 0.9, chunk_bytes=cb)
    got = replica.numpy()[pidx]
    assert np.array_equal(got.view(np.uint32), ref_w.view(np.uint32)), f"rank {rank}: replica"
    # every chunk's owner range is a whole number of chunks, ranges abut and cover
    assert ranges[0][0] == 0 and ranges[-1][1] == Ep
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank}/{world} ok: owned [{b},{e}) sends {plan.nvlink_bytes_out()} B")


if __name__ == "__main__":
    main()
