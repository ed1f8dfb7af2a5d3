"""The library's fused kernel timed through the ctypes binding WITHOUT torch
(argv[1] == "notorch") or after `import torch` + CUDA init ("torch"): the
same sequence as scripts/flat_c_probe.c (VGG-19-sized single key, 8 BORROW
pushes of cudaMalloc'd buffers, 30 rounds after 10 warm-up, L2 policy argv[2]).
Timing with cudart events through ctypes."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
mode, cache = sys.argv[1], int(sys.argv[2])
if mode == "torch":
    import torch
    torch.cuda.init()
    torch.zeros(1, device="cuda:0")
from paper_1805_07891_b200 import capi  # noqa: E402

rt = C.CDLL("/usr/local/cuda/lib64/libcudart.so.12")
E = 143667264
cfg = capi.phub_config_default()
keys = (C.c_uint64 * 1)(E)
cfg.key_num_elements = keys
cfg.num_keys = 1
cfg.num_workers = 8
ctx = capi.phub_init(cfg)
capi.phub_set_option(ctx, capi.PHUB_OPT_CACHE, cache)
g = [capi.phub_alloc_shared(0, 4 * E) for _ in range(8)]
for p in g:
    rt.cudaMemset(C.c_void_p(p), 0, C.c_size_t(4 * E))
a, b = C.c_void_p(), C.c_void_p()
rt.cudaEventCreate(C.byref(a))
rt.cudaEventCreate(C.byref(b))
for r in range(40):
    if r == 10:
        rt.cudaEventRecord(a, None)
    for w in range(8):
        capi.phub_push(ctx, w, capi.PHUB_ALL_KEYS, g[w], E, capi.PHUB_BORROW)
    capi.phub_aggregate_optimize(ctx)
rt.cudaEventRecord(b, None)
rt.cudaEventSynchronize(b)
ms = C.c_float()
rt.cudaEventElapsedTime(C.byref(ms), a, b)
print(json.dumps({"harness": f"python-{mode}", "cache": cache, "ms": round(ms.value / 30, 4)}))
