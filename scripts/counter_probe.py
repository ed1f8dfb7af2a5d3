"""Probe (scratch evidence): which NVML NVLink byte counters are readable on
this box, with which scope, and do they agree with a known 4 GiB peer copy?
One process, 2 GPUs."""
import json
import time

import pynvml as nv
import torch

nv.nvmlInit()
FIELDS = {"THROUGHPUT_DATA_TX": 138, "THROUGHPUT_DATA_RX": 139, "THROUGHPUT_RAW_TX": 140,
          "THROUGHPUT_RAW_RX": 141, "COUNT_XMIT_BYTES": 202, "COUNT_RCV_BYTES": 204}
hs = [nv.nvmlDeviceGetHandleByIndex(i) for i in range(torch.cuda.device_count())]


def read(h, scopes):
    req = [(fid, sc) for fid in FIELDS.values() for sc in scopes]
    vals = nv.nvmlDeviceGetFieldValues(h, req)
    out = {}
    for (fid, sc), v in zip(req, vals):
        name = [k for k, x in FIELDS.items() if x == fid][0]
        out[f"{name}@{sc}"] = (int(v.nvmlReturn), int(v.value.ullVal), int(v.valueType))
    return out


scopes = list(range(18)) + [0xFFFFFFFF]
b0 = read(hs[0], scopes)
print("returns:", {k: v[0] for k, v in b0.items() if k.endswith("@0") or k.endswith("@4294967295")})
n = 1 << 28
a = torch.ones(n, device="cuda:0")
b = torch.empty(n, device="cuda:1")
torch.cuda.synchronize()
before = [read(h, scopes) for h in hs[:2]]
for _ in range(4):
    b.copy_(a)                      # 4 GiB GPU0 -> GPU1 (copy engine over NVLink)
torch.cuda.synchronize()
time.sleep(1.5)
after = [read(h, scopes) for h in hs[:2]]
for g in range(2):
    d = {k: after[g][k][1] - before[g][k][1] for k in after[g]
         if after[g][k][0] == 0 and after[g][k][1] != before[g][k][1]}
    print(f"gpu{g} changed counters (4 GiB 0->1):", json.dumps(d))
print("valueType of ok fields:", {k: v[2] for k, v in b0.items() if v[0] == 0})
