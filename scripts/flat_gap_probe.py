"""Why does the library's fused kernel run ~4 % slower in bench.py than the same
arithmetic in a standalone CUDA program (scripts/flat_variants.cu)?  Times
phub_aggregate_optimize on VGG-19 (N = 8) back to back, varying one thing at
a time: gradient buffers from torch's allocator vs cudaMalloc
(phub_alloc_shared); events around every launch vs around the whole loop;
L2 policy bypass vs resident.  Mean ms of 30 launches after 10 warm-up."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1805_07891_b200 import PHub, capi  # noqa: E402
from paper_1805_07891_b200.phub import _CudaArray  # noqa: E402
from workloads import grad_stream, manifest  # noqa: E402
from workloads.generate import values_torch  # noqa: E402


def run(alloc, per_launch_events, cache, N=8):
    dev = torch.device("cuda:0")
    sizes = manifest("vgg19")
    hub = PHub(sizes, N, device=0)
    hub.set_option(capi.PHUB_OPT_CACHE, cache)
    E, Ep = hub.E, hub.E_padded
    idx = torch.as_tensor(hub.padded_index(), device=dev)
    hub.load_state(values_torch(1, 0, E, 20, dev), values_torch(2, 0, E, 25, dev))
    grads, raw = [], []
    for w in range(N):
        if alloc == "torch":
            b = torch.zeros(Ep, dtype=torch.float32, device=dev)
        else:
            p = capi.phub_alloc_shared(0, 4 * Ep)
            raw.append(p)
            b = torch.as_tensor(_CudaArray(p, Ep, hub), device=dev)
            b.zero_()
        b[idx] = values_torch(grad_stream(w), 0, E, 25, dev)
        grads.append(b)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()

    def one():
        for w in range(N):
            hub.push(w, grads[w])
        hub.aggregate_optimize()

    for _ in range(10):
        one()
    torch.cuda.synchronize()
    if per_launch_events:
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(30)]
        for a, b in ev:
            for w in range(N):
                hub.push(w, grads[w])
            a.record(s)
            hub.aggregate_optimize()
            b.record(s)
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in ev) / 30
    else:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(30):
            one()
        b.record(s)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 30
    ptrs = [g.data_ptr() % (2 << 20) for g in grads]
    hub.close()
    del grads
    for p in raw:
        capi.phub_free_shared(0, p)
    torch.cuda.empty_cache()
    return ms, ptrs


if __name__ == "__main__":
    alloc, ple, cache = sys.argv[1], sys.argv[2] == "1", int(sys.argv[3])
    ms, ptrs = run(alloc, ple, cache)
    print(json.dumps({"alloc": alloc, "per_launch_events": ple, "cache": cache, "ms": round(ms, 4),
                      "grad_offsets_mod_2MiB": ptrs}))
