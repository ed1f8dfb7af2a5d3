"""Per-item timeline of the scheduled exchange (diagnostic).

    torchrun --nproc-per-node G scripts/sched_trace.py OUT_DIR [lag] [block] [consumers]

Runs SchedShardedPHub on VGG-19 (8 workers), 5 rounds, with PHUB_OPT_SCHED_TRACE
set: every item of the last round records when its ticket was taken, when its
wait finished and when it was done (%globaltimer ns) and which CTA / SM ran it.
Each rank saves OUT_DIR/trace_rank{r}.npz (items in lane order + times);
analyse with scripts/sched_trace_report.py.
"""
import datetime
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1805_07891_b200 import capi  # noqa: E402
from paper_1805_07891_b200.sharded import SchedShardedPHub  # noqa: E402
from workloads import manifest  # noqa: E402


def main():
    out = sys.argv[1]
    lag = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    block = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
    cons = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    os.makedirs(out, exist_ok=True)
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=300))
    rank, G = dist.get_rank(), dist.get_world_size()
    sizes = manifest("vgg19")
    sh = SchedShardedPHub(sizes, 8, device=local, block=block, lag=lag, consumer_ctas=cons)
    items, _nf = capi.phub_sched_plan(G, rank, sh.W, sh.bounds, sh.split, block, lag, sh.taper)
    items = list(items)
    cons_t = (capi.PHUB_ITEM_CONSUME_RAW, capi.PHUB_ITEM_CONSUME_FINAL)
    lanes = [it for it in items if it.type not in cons_t] + [it for it in items if it.type in cons_t]
    tr = torch.zeros(4 * len(lanes), dtype=torch.int64, device=dev)
    sh.hub.set_option(capi.PHUB_OPT_SCHED_TRACE, tr.data_ptr())
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for r in range(5):
        if r == 4:
            ev[0].record()
        sh.exchange()
        if r == 4:
            ev[1].record()
    torch.cuda.synchronize()
    sh.check()
    t = tr.cpu().numpy().reshape(-1, 4)
    np.savez(os.path.join(out, f"trace_rank{rank}.npz"), t=t,
             lo=np.array([it.lo for it in lanes]), hi=np.array([it.hi for it in lanes]),
             type=np.array([it.type for it in lanes]), dst=np.array([it.dst for it in lanes]),
             bounds=np.array(sh.bounds), split=np.array(sh.split),
             ms=ev[0].elapsed_time(ev[1]), lag=lag, block=block)
    print(f"rank {rank}: {len(lanes)} items, round {ev[0].elapsed_time(ev[1]):.3f} ms")
    sh.hub.set_option(capi.PHUB_OPT_SCHED_TRACE, 0)
    sh.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
