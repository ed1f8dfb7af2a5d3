"""Multi-GPU parity worker (torchrun, NCCL): the sharded exchanges vs the CPU oracle.

Each rank hosts N/G workers; after R rounds every rank's full replica must
equal R oracle rounds bit for bit (full-mantissa inputs: a wrong summation
order fails).  mode "allreduce" is the NEGATIVE CONTROL (AllReduceBaseline:
NCCL all-reduce, then Nesterov everywhere): it must be within rounding of the
oracle but NOT bit-exact -- proving the exact exchanges' parity is evidence of
the worker-order sum.
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
    AllReduceBaseline, ChainShardedPHub, P2PShardedPHub, PushShardedPHub, SchedShardedPHub,
    ShardedPHub)
from workloads import grad_stream, manifest  # noqa: E402
from workloads.generate import fullmant_np, fullmant_torch  # noqa: E402


def main():
    name, N, cb, rounds = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    mode = sys.argv[5] if len(sys.argv) > 5 else "nccl"
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=300))
    rank, G = dist.get_rank(), dist.get_world_size()
    special = {"small": [3, 3, 9408, 64, 64, 4096, 20000, 1000, 7], "one": [5]}
    sizes = special[name] if name in special else manifest(name)
    E = sum(sizes)
    if mode.startswith("chain"):
        # chain: block-streaming flags; chain_flags / chain_barrier: per piece
        sync = {"chain": "blocks", "chain_flags": "flags", "chain_barrier": "barrier"}[mode]
        sh = ChainShardedPHub(sizes, N, chunk_size_bytes=cb, device=local, pieces=3, sync=sync,
                              block=2048)
    elif mode == "push":
        sh = PushShardedPHub(sizes, N, chunk_size_bytes=cb, device=local, block=2048)
    elif mode == "sched":
        sh = SchedShardedPHub(sizes, N, chunk_size_bytes=cb, device=local, block=2048, lag=1)
    elif mode == "sched_raw":        # the G = 8 plan (all RAW, one lane) at any G
        sh = SchedShardedPHub(sizes, N, chunk_size_bytes=cb, device=local, block=2048,
                              weights=[1.0 / G] * G, raw_frac=[1.0] * G)
    elif mode == "allreduce":
        sh = AllReduceBaseline(sizes, N, chunk_size_bytes=cb, device=local)
    else:
        cls = P2PShardedPHub if mode == "p2p" else ShardedPHub
        sh = cls(sizes, N, chunk_size_bytes=cb, device=local)
    fused = mode in ("p2p", "push", "sched", "sched_raw") or mode.startswith("chain")
    w_ref, v_ref = fullmant_np(1, 0, E), fullmant_np(2, 0, E)
    sh.hub.load_state(w_ref, v_ref)
    idx = torch.as_tensor(sh.hub.padded_index(), device=dev)
    for r in range(rounds):
        grads = sh.gradients() if fused else {}
        for w in sh.hosted:
            b = grads[w] if fused else torch.empty(sh.hub.E_padded, device=dev)
            b.fill_(float("nan"))
            b[idx] = fullmant_torch(grad_stream(w) + 37 * r, 0, E, dev)
            grads[w] = b
        if fused:
            sh.exchange()
        else:
            sh.exchange(grads)
        hg = [fullmant_np(grad_stream(w) + 37 * r, 0, E) for w in range(N)]
        w_ref, v_ref, _ = oracle.round_(sizes, hg, w_ref, v_ref, 0.1, 0.9, chunk_bytes=cb)
    torch.cuda.synchronize()
    if mode.startswith("chain") or mode in ("push", "sched", "sched_raw"):
        sh.check()                   # collective: raises on every rank if a device wait expired
    got = sh.weights()[idx].cpu().numpy()
    bad = int(np.sum(got.view(np.uint32) != w_ref.view(np.uint32)))
    if mode == "allreduce":          # negative control: within rounding, NOT bit-exact
        rel = np.abs(got.astype(np.float64) - w_ref) / np.maximum(np.abs(w_ref.astype(np.float64)),
                                                                 1e-30)
        ok = bad > 0.01 * E and float(np.median(rel)) < 1e-6
        print(f"rank {rank}: allreduce differs on {bad}/{E} elements, median rel "
              f"{float(np.median(rel)):.2e}")
    else:
        ok = bad == 0
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    sh.close()
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank}/{G}: {'ok' if ok else f'MISMATCH {bad} elements'}")
    sys.exit(0 if flag.item() == 0 else 1)


if __name__ == "__main__":
    main()
