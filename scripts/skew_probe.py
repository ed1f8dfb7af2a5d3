"""Placement probe for the 1-GPU fused kernel (DRAM channel/bank aliasing):
times phub_aggregate_optimize on VGG-19 x 8 workers with the 8 gradient
buffers placed (a) as separate allocations, (b) in one allocation at stride
E_padded + skew for several skews.  Same kernel, same bytes; only the
relative addresses of the N + 2 streams change.

    python scripts/skew_probe.py > gpurun_out/skew.json
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1805_07891_b200 import PHub, capi  # noqa: E402
from workloads import grad_stream, manifest  # noqa: E402
from workloads.generate import values_torch  # noqa: E402


def time_hub(hub, grads, steps=40, warmup=5):
    batch = [(w, capi.PHUB_ALL_KEYS, g) for w, g in enumerate(grads)]
    for _ in range(warmup):
        hub.push_batch(batch)
        hub.aggregate_optimize()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    for a, b in ev:
        hub.push_batch(batch)
        a.record()
        hub.aggregate_optimize()
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)
    return ms[len(ms) // 2], ms[0]


def main():
    dev = torch.device("cuda:0")
    sizes = manifest("vgg19")
    N = 8
    hub = PHub(sizes, N, device=0)
    E, Ep = hub.E, hub.E_padded
    hub.load_state(values_torch(1, 0, E, 20, dev), values_torch(2, 0, E, 25, dev))
    src = values_torch(grad_stream(0), 0, Ep, 25, dev)
    out = []
    sep = [src.clone() for _ in range(N)]
    med, mn = time_hub(hub, sep)
    out.append({"placement": "separate allocations", "ms_median": med, "ms_min": mn})
    del sep
    torch.cuda.empty_cache()
    for skew in (0, 512, 2048, 8192, 33 * 1024 // 4, 256 * 1024, 1 << 20, (1 << 20) + 8192):
        stride = Ep + skew
        big = torch.empty(N * stride + 64, dtype=torch.float32, device=dev)
        grads = []
        for w in range(N):
            g = big[w * stride: w * stride + Ep]
            g.copy_(src)
            grads.append(g)
        med, mn = time_hub(hub, grads)
        out.append({"placement": f"one allocation, stride E_padded + {skew} elements",
                    "ms_median": med, "ms_min": mn})
        del grads, big
        torch.cuda.empty_cache()
    bytes_ = (4 * N + 16) * hub.owned_elements()
    for r in out:
        r["GBps"] = round(bytes_ / (r["ms_median"] / 1e3) / 1e9, 1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
