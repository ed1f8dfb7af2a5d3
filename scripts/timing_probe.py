"""Scratch probe: does bracketing every launch with CUDA events change the
fused kernel's time?  VGG-19, N = 8, both L2 policies, alternating orders."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1805_07891_b200 import PHub, capi  # noqa: E402
from workloads import manifest  # noqa: E402

dev = torch.device("cuda:0")
sizes = manifest("vgg19")
hub = PHub(sizes, 8, device=0)
grads = [torch.zeros(hub.E_padded, device=dev) for _ in range(8)]
if "--random" in sys.argv:                         # bench.py's inputs
    from workloads import grad_stream
    from workloads.generate import values_torch
    idx = torch.as_tensor(hub.padded_index(), device=dev)
    hub.load_state(values_torch(1, 0, hub.E, 20, dev), values_torch(2, 0, hub.E, 25, dev))
    for w in range(8):
        grads[w][idx] = values_torch(grad_stream(w), 0, hub.E, 25, dev)
    torch.cuda.synchronize()
batch = [(w, capi.PHUB_ALL_KEYS, grads[w]) for w in range(8)]
st = torch.cuda.current_stream(dev)


def step():
    hub.push_batch(batch)
    hub.aggregate_optimize()


def back_to_back(reps=20):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        step()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def per_event(reps=20):
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for i in range(reps):
        hub.push_batch(batch)
        ev[i][0].record(st)
        hub.aggregate_optimize()
        ev[i][1].record(st)
    b.record(st)
    torch.cuda.synchronize()
    return sum(x.elapsed_time(y) for x, y in ev) / reps, a.elapsed_time(b) / reps


if "--sampler" in sys.argv:                        # bench.py's NVML clock sampler on/off
    from bench import ClockSampler
    for phase in ("off", "on", "off", "on"):
        cs = ClockSampler(0) if phase == "on" else None
        if cs:
            cs.start()
        for trial in range(3):
            k, tot = per_event()
            print(json.dumps({"sampler": phase, "trial": trial, "per_event_kernel_ms": round(k, 4),
                              "per_event_total_ms": round(tot, 4)}))
        if cs:
            cs.stop()
            print(json.dumps({"sampler_summary": cs.summary()}))
    sys.exit(0)

for pol in ("BYPASS", "ENABLED", "BYPASS"):
    hub.set_option(capi.PHUB_OPT_CACHE, getattr(capi, f"PHUB_CACHE_{pol}"))
    for _ in range(5):
        step()
    for trial in range(3):
        k, tot = per_event()
        bb = back_to_back()
        k2, tot2 = per_event()
        print(json.dumps({"policy": pol, "trial": trial, "per_event_kernel_ms": round(k, 4),
                          "per_event_total_ms": round(tot, 4), "back_to_back_ms": round(bb, 4),
                          "per_event_again_kernel_ms": round(k2, 4),
                          "per_event_again_total_ms": round(tot2, 4)}))
