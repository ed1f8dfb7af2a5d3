"""Multi-GPU parity worker for the hierarchical reduction (torchrun, NCCL;
SURVEY 8(f) NEXT-4): every GPU is one rack with P local
workers; after `rounds` rounds every rank's replica must equal the oracle's
hierarchical rounds (oracle.hier_round) bit for bit -- the whole model for
small manifests, sampled elements (oracle.hier_elems) for full-size ones.

    torchrun --nproc-per-node G hier_exchange_worker.py NAME P CHUNK_BYTES ROUNDS BLOCK
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
from paper_1805_07891_b200.sharded import HierPHub  # noqa: E402
from workloads import grad_stream, manifest  # noqa: E402
from workloads.generate import fullmant_at_np, fullmant_np, fullmant_torch  # noqa: E402

SPECIAL = {"small": [3, 3, 9408, 64, 64, 4096, 20000, 1000, 7], "one": [5]}
SAMPLED = ("vgg19", "alexnet", "resnet269")


def main():
    name, P, cb, rounds = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    block = int(sys.argv[5]) if len(sys.argv) > 5 else 2048
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=300))
    rack, R = dist.get_rank(), dist.get_world_size()
    sizes = SPECIAL[name] if name in SPECIAL else manifest(name)
    E = sum(sizes)
    sh = HierPHub(sizes, workers_per_rack=P, chunk_size_bytes=cb, device=local, block=block)
    hub = sh.hub
    idx = torch.as_tensor(hub.padded_index(), device=dev)
    hub.load_state(fullmant_torch(1, 0, E, dev), fullmant_torch(2, 0, E, dev))

    def stream(r, k, rnd):                     # worker k of rack r, round rnd
        return grad_stream(r * P + k) + 37 * rnd

    for rnd in range(rounds):
        g = sh.gradients(slot=rnd % 2)
        for k in range(P):
            g[k].fill_(float("nan"))
            g[k][idx] = fullmant_torch(stream(rack, k, rnd), 0, E, dev)
        sh.exchange(slot=rnd % 2)
    torch.cuda.synchronize()
    if name in SAMPLED:
        rng = np.random.default_rng(11 + rack)
        starts = np.concatenate([[0], np.cumsum(sizes)])
        samp = np.unique(np.concatenate([rng.integers(0, E, 20000), starts[:-1],
                                         starts[1:] - 1])).astype(np.int64)
        got = sh.weights()[idx[torch.as_tensor(samp, device=dev)]].cpu().numpy()
        w_ref, v_ref = fullmant_at_np(1, samp), fullmant_at_np(2, samp)
        for rnd in range(rounds):
            gs = np.stack([np.stack([fullmant_at_np(stream(r, k, rnd), samp) for k in range(P)])
                           for r in range(R)])
            w_ref, v_ref, _ = oracle.hier_elems(gs, w_ref, v_ref, 0.1, 0.9)
    else:
        got = sh.weights()[idx].cpu().numpy()
        w_ref, v_ref = fullmant_np(1, 0, E), fullmant_np(2, 0, E)
        w_flat, v_flat = w_ref, v_ref
        for rnd in range(rounds):
            racks = [[fullmant_np(stream(r, k, rnd), 0, E) for k in range(P)] for r in range(R)]
            w_ref, v_ref, _ = oracle.hier_round(sizes, racks, w_ref, v_ref, 0.1, 0.9,
                                                chunk_bytes=cb)
            w_flat, v_flat, _ = oracle.round_(sizes, [g for rk in racks for g in rk], w_flat,
                                              v_flat, 0.1, 0.9, chunk_bytes=cb)
        if P > 1 and E > 100:        # rack grouping must be visible (else parity proves nothing)
            diff = int(np.sum(got.view(np.uint32) != w_flat.view(np.uint32)))
            print(f"rank {rack}: hierarchical differs from the flat worker order on {diff}/{E}")
            assert diff > 0
    sh.check()                       # collective: raises on every rank if a device wait expired
    ok = np.array_equal(got.view(np.uint32), w_ref.view(np.uint32))
    bad = int(np.sum(got.view(np.uint32) != w_ref.view(np.uint32)))
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    sh.close()
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rack}/{R}: {'ok' if ok else f'MISMATCH {bad} elements'}")
    sys.exit(0 if flag.item() == 0 else 1)


if __name__ == "__main__":
    main()
