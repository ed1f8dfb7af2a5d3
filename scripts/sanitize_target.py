"""Small single-GPU workload touching every kernel (flat 256/128-bit one-shot
and persistent, chunk tiles with ragged tails, bulk-copy ring, wide ablation,
partial sum + flag-ordered range aggregate) -- the target of compute-sanitizer
runs.  Exits non-zero on any parity mismatch vs the oracle."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1805_07891_b200 import PHub, capi  # noqa: E402
from workloads import grad_stream, values_np  # noqa: E402

SIZES = [3, 3, 9408, 64, 64, 4096, 20000, 1000, 7]
E = sum(SIZES)
DEV = "cuda:0"


def grads(hub, n):
    idx = torch.as_tensor(hub.padded_index(), device=DEV)
    out = []
    for w in range(n):
        b = torch.zeros(hub.E_padded, device=DEV)
        b[idx] = torch.as_tensor(values_np(grad_stream(w), 0, E, 25), device=DEV)
        out.append(b)
    return out


def main():
    w0, v0 = values_np(1, 0, E, 20), values_np(2, 0, E, 25)
    hg = [values_np(grad_stream(w), 0, E, 25) for w in range(4)]
    rw, _, _ = oracle.round_(SIZES, hg, w0, v0, 0.1, 0.9)
    bad = 0
    variants = [("flat", capi.PHUB_KERNEL_FLAT, {}), ("flat128", capi.PHUB_KERNEL_FLAT128, {}),
                ("persistent", capi.PHUB_KERNEL_FLAT, {capi.PHUB_OPT_FLAT_ONESHOT: 0}),
                ("tiles", capi.PHUB_KERNEL_TILES, {capi.PHUB_OPT_TILE_ELEMS: 100}),
                ("bulk", capi.PHUB_KERNEL_BULK, {}), ("wide", capi.PHUB_KERNEL_WIDE, {})]
    for name, kern, opts in variants:
        hub = PHub(SIZES, 4, device=0, keep_aggregate=True)
        hub.load_state(w0, v0)
        hub.set_option(capi.PHUB_OPT_KERNEL, kern)
        for k, v in opts.items():
            hub.set_option(k, v)
        for w, g in enumerate(grads(hub, 4)):
            hub.push(w, g)
        hub.aggregate_optimize()
        w, _, _ = hub.read_state()
        ok = np.array_equal(w.view(np.uint32), rw.view(np.uint32))
        bad += not ok
        print(name, "ok" if ok else "MISMATCH")
        hub.close()
    # chain building blocks with device flags
    head = PHub(SIZES, 2, device=0)
    gd = grads(head, 4)
    part = torch.empty(head.E_padded, device=DEV)
    flags = torch.zeros(2, dtype=torch.int32, device=DEV)
    st = head._stream(None)
    capi.phub_partial_sum(head.ctx, [g.data_ptr() for g in gd[:2]], part.data_ptr(), 0,
                          head.E_padded, st, signal=(flags.data_ptr(), 1))
    tail = PHub(SIZES, 3, device=0, rescale=0.25)
    tail.load_state(w0, v0)
    tail.push(0, part)
    tail.push(1, gd[2])
    tail.push(2, gd[3])
    capi.phub_aggregate_range(tail.ctx, 0, tail.E_padded, st, wait=(flags.data_ptr(), 1))
    w, _, _ = tail.read_state()
    ok = np.array_equal(w.view(np.uint32), rw.view(np.uint32)) and \
        capi.phub_sync_timeouts(tail.ctx) == 0
    bad += not ok
    print("chain", "ok" if ok else "MISMATCH")
    head.close()
    tail.close()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
