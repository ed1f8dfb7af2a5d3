"""The chained exchange's two block-streamed kernels on ONE GPU, back to back
on one stream (producer first, so no kernel waits on a co-resident one), at
full VGG-19 size: k_blocks<4, partial> over workers 0..3, then
k_blocks<5, fused Nesterov> over the partial + workers 4..7 -- for ncu
(`-k regex:k_blocks`), which cannot profile the 2-rank run.  Prints the
per-kernel times (CUDA events) and checks sampled outputs against the oracle.

    python scripts/chain_one_gpu.py [--block 12288] [--rounds 3]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1805_07891_b200 import PHub, capi  # noqa: E402
from workloads import grad_stream, manifest  # noqa: E402
from workloads.generate import values_at_np, values_torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--block", type=int, default=12288)
    ap.add_argument("--rounds", type=int, default=3)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    sizes = manifest("vgg19")
    E = sum(sizes)
    head = PHub(sizes, 4, device=0)
    tail = PHub(sizes, 5, device=0, rescale=1.0 / 8)
    Ep = head.E_padded
    idx = torch.as_tensor(head.padded_index(), device=dev)
    tail.load_state(values_torch(1, 0, E, 20, dev), values_torch(2, 0, E, 25, dev))
    g = []
    for w in range(8):
        b = torch.zeros(Ep, device=dev)
        b[idx] = values_torch(grad_stream(w), 0, E, 25, dev)
        g.append(b)
    part = torch.empty(Ep, device=dev)
    nblk = -(-Ep // args.block)
    flags = torch.zeros(nblk, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream(dev)
    t = []
    for r in range(1, args.rounds + 1):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(st)
        capi.phub_partial_sum(head.ctx, [x.data_ptr() for x in g[:4]], part.data_ptr(), 0, Ep,
                              st.cuda_stream, signal=(flags.data_ptr(), r), block=args.block)
        e1.record(st)
        tail.push(0, part)
        for k in range(4):
            tail.push(1 + k, g[4 + k])
        capi.phub_aggregate_range(tail.ctx, 0, Ep, st.cuda_stream, wait=(flags.data_ptr(), r),
                                  block=args.block)
        e2.record(st)
        torch.cuda.synchronize()
        t.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
    assert capi.phub_sync_timeouts(tail.ctx) == 0
    # sampled check of the last round's w' against the oracle (3 rounds of the same grads)
    import oracle
    rng = np.random.default_rng(5)
    samp = np.unique(rng.integers(0, E, 4000)).astype(np.int64)
    w_ref, v_ref = values_at_np(1, samp, 20), values_at_np(2, samp, 25)
    gs = np.stack([values_at_np(grad_stream(w), samp, 25) for w in range(8)])
    for _ in range(args.rounds):
        w_ref, v_ref, _ = oracle.elems(gs, w_ref, v_ref, 0.1, 0.9)
    w_all, _, _ = tail.read_state()
    ok = np.array_equal(w_all[samp].view(np.uint32), w_ref.view(np.uint32))
    prod = min(a for a, _ in t)
    cons = min(b for _, b in t)
    print(f"block {args.block}: producer (4 workers -> partial) {prod:.3f} ms = "
          f"{20 * E / prod / 1e6:.0f} GB/s; consumer (partial + 4 workers + NAG) {cons:.3f} ms = "
          f"{36 * E / cons / 1e6:.0f} GB/s; sampled w' {'bit-exact' if ok else 'MISMATCH'}")
    head.close()
    tail.close()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
