"""Full-size multi-GPU parity worker (torchrun, NCCL): the exchange bench.py
times at N > 1 (`--mode auto`: the scheduled exchange), at BASELINE.json's full model size,
checked against the CPU oracle on sampled elements (the oracle computes them
one by one from independently generated inputs).

    torchrun --nproc-per-node G full_size_exchange_worker.py vgg19 [mode] [rounds]

Every rank's pulled replica is checked at key starts/ends, chunk boundaries,
owner-range and block boundaries and random elements.
"""
import datetime
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1805_07891_b200.sharded import (  # noqa: E402
    ChainShardedPHub, P2PShardedPHub, PushShardedPHub, SchedShardedPHub)
from workloads import grad_stream, manifest  # noqa: E402
from workloads.generate import fullmant_at_np, fullmant_np, fullmant_torch  # noqa: E402


def sample(sizes, E, ranges, block, rng):
    """Real-element indices: key starts/ends, 32 KB chunk starts, the elements
    around owner-range and block boundaries (mapped back from the padded
    layout), and 20000 random ones."""
    starts = np.concatenate([[0], np.cumsum(sizes)])
    pts = [rng.integers(0, E, 20000), starts[:-1], starts[1:] - 1]
    for k in range(len(sizes)):
        pts.append(np.arange(starts[k], starts[k + 1], 8192)[:32])
    return np.unique(np.concatenate(pts)).astype(np.int64)


def main():
    name = sys.argv[1]
    mode = sys.argv[2] if len(sys.argv) > 2 else "auto"
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    N, cb = 8, 32768
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=300))
    rank, G = dist.get_rank(), dist.get_world_size()
    if mode == "auto":                       # bench.py --mode auto
        mode = "sched"
    sizes = manifest(name)
    E = sum(sizes)
    cls = {"chain": ChainShardedPHub, "p2p": P2PShardedPHub, "push": PushShardedPHub,
           "sched": SchedShardedPHub}[mode]
    sh = cls(sizes, N, chunk_size_bytes=cb, device=local)
    hub = sh.hub
    idx = torch.as_tensor(hub.padded_index(), device=dev)
    hub.load_state(fullmant_torch(1, 0, E, dev), fullmant_torch(2, 0, E, dev))
    for r in range(rounds):
        g = sh.gradients(slot=r % 2)
        for w in sh.hosted:
            g[w].fill_(float("nan"))
            g[w][idx] = fullmant_torch(grad_stream(w) + 37 * r, 0, E, dev)
        sh.exchange(slot=r % 2)
    torch.cuda.synchronize()
    rng = np.random.default_rng(7 + rank)
    samp = sample(sizes, E, None, None, rng)
    got = sh.weights()[idx[torch.as_tensor(samp, device=dev)]].cpu().numpy()
    w_ref = fullmant_at_np(1, samp)
    v_ref = fullmant_at_np(2, samp)
    for r in range(rounds):
        gs = np.stack([fullmant_at_np(grad_stream(w) + 37 * r, samp) for w in range(N)])
        w_ref, v_ref, _ = oracle.elems(gs, w_ref, v_ref, 0.1, 0.9)
    if mode in ("chain", "push", "sched"):
        sh.check()                   # collective: raises on every rank if a device wait expired
    ok = np.array_equal(got.view(np.uint32), w_ref.view(np.uint32))
    bad = int(np.sum(got.view(np.uint32) != w_ref.view(np.uint32)))
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    sh.close()
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank}/{G} {name} {mode} {samp.size} sampled: "
          f"{'ok' if ok else f'MISMATCH {bad} elements'}")
    sys.exit(0 if flag.item() == 0 else 1)


if __name__ == "__main__":
    main()
