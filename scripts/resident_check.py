"""Is the resident slice of w really in L2 after a round?  (No profiler: ncu's
own activity between launches disturbs L2.)  After each of 10 rounds of the
fused kernel (VGG-19, N = 8), time a read of 32 MiB of w with CUDA events --
the kept slice (the last 32 MiB of the owned range) or the first 32 MiB --
under the resident and the bypass policy.  An L2-resident 32 MiB reads in a
few us; from HBM it takes >= 32 MiB / 6.5 TB/s = 5.2 us plus launch."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1805_07891_b200 import PHub, capi  # noqa: E402
from workloads import grad_stream, manifest  # noqa: E402
from workloads.generate import values_torch  # noqa: E402


def main(cache):
    dev = torch.device("cuda:0")
    sizes = manifest("vgg19")
    N = 8
    hub = PHub(sizes, N, device=0)
    hub.set_option(capi.PHUB_OPT_CACHE, cache)
    E, Ep = hub.E, hub.E_padded
    idx = torch.as_tensor(hub.padded_index(), device=dev)
    hub.load_state(values_torch(1, 0, E, 20, dev), values_torch(2, 0, E, 25, dev))
    grads = []
    for w in range(N):
        b = torch.zeros(Ep, device=dev)
        b[idx] = values_torch(grad_stream(w), 0, E, 25, dev)
        grads.append(b)
    del idx
    w = hub.weights()
    n = (32 << 20) // 4
    out = torch.empty(1, device=dev)
    res = {"tail": [], "head": []}
    for r in range(30):
        for k in range(N):
            hub.push(k, grads[k])
        hub.aggregate_optimize()
        if r < 10:
            continue
        which = "tail" if r % 2 else "head"
        sl = w[Ep - n:] if which == "tail" else w[:n]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        torch.sum(sl, dim=0, out=out[0])
        b.record()
        torch.cuda.synchronize()
        res[which].append(a.elapsed_time(b) * 1e3)
    hub.close()
    return {k: round(sorted(v)[len(v) // 2], 2) for k, v in res.items()}


if __name__ == "__main__":
    for cache, name in ((capi.PHUB_CACHE_RESIDENT, "resident"), (capi.PHUB_CACHE_BYPASS, "bypass")):
        print(json.dumps({"policy": name, "median_us_read_32MiB": main(cache)}))
