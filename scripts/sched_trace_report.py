"""Summarise scripts/sched_trace.py output: per rank and item type, the time
items spent waiting vs working, the busy CTAs over time, and when each rank's
lanes finished (relative to the rank's first ticket of the round: the GPUs' %globaltimer
clocks are not aligned, so ranks are not compared in absolute time).

    python scripts/sched_trace_report.py DIR
"""
import glob
import sys

import numpy as np

NAMES = {1: "RAW_PUSH", 2: "CHAIN", 3: "CONSUME_RAW", 4: "CONSUME_FINAL"}


def main():
    files = sorted(glob.glob(f"{sys.argv[1]}/trace_rank*.npz"))
    data = [np.load(f) for f in files]
    for r, d in enumerate(data):
        t = d["t"].astype(np.int64)
        ok = t[:, 0] > 0
        t0 = int(t[ok, 0].min())       # per rank: the GPUs' %globaltimer clocks are not aligned
        print(f"rank {r}: round {float(d['ms']):.3f} ms, {ok.sum()} items")
        for ty in (1, 2, 3, 4):
            m = ok & (d["type"] == ty)
            if not m.any():
                continue
            wait = (t[m, 1] - t[m, 0]) / 1e3
            work = (t[m, 2] - t[m, 1]) / 1e3
            el = (d["hi"][m] - d["lo"][m]).sum()
            print(f"  {NAMES[ty]:14s} n={m.sum():5d} elems={el / 1e6:7.2f}M  wait us "
                  f"mean {wait.mean():7.1f} p90 {np.percentile(wait, 90):7.1f}  work us mean "
                  f"{work.mean():6.1f}  first {(t[m, 0].min() - t0) / 1e3:7.1f} "
                  f"last done {(t[m, 2].max() - t0) / 1e3:7.1f}")
        # busy CTAs (working, not waiting) in 100-us bins
        end = (t[ok, 2].max() - t0) / 1e3
        bins = np.arange(0, end + 100, 100)
        busy = np.zeros(len(bins))
        waiting = np.zeros(len(bins))
        for a, b, c in zip((t[ok, 0] - t0) / 1e3, (t[ok, 1] - t0) / 1e3, (t[ok, 2] - t0) / 1e3):
            waiting[int(a // 100):int(b // 100) + 1] += 1
            busy[int(b // 100):int(c // 100) + 1] += 1
        print("  per 100us bin: working items", busy.astype(int).tolist()[:40])
        print("                 waiting items", waiting.astype(int).tolist()[:40])


if __name__ == "__main__":
    main()
