"""Collect bench.py JSON lines into one CSV with a fixed schema (SURVEY 5,
"a CSV row per (config, G, chunk size, variant) with the 8(d) fields";
SPEC's bench-harness idea of a stable header).

    python scripts/results_csv.py profiles > profiles/results_r01.csv

Every *.json file under the given directories is scanned for lines that are
bench.py output (a JSON object with "metric" and "value"); one row each.
"""
import csv
import glob
import json
import os
import sys

COLUMNS = ["file", "impl", "workload", "n_gpus", "workers", "chunk_bytes", "mode", "kernel",
           "value_GBps", "ms_per_step", "exchanges_per_s", "scaling", "roofline_bound",
           "roofline_achieved", "roofline_peak", "roofline_frac", "nvlink_frac",
           "owner_phase_GBps", "e2e_GBps", "sm_mhz", "throttle_reasons"]


def rows(paths):
    for root in paths:
        for f in sorted(glob.glob(os.path.join(root, "**", "*.json"), recursive=True)):
            try:
                lines = open(f).read().splitlines()
            except OSError:
                continue
            for ln in lines:
                ln = ln.strip()
                if not ln.startswith("{"):
                    continue
                try:
                    d = json.loads(ln)
                except ValueError:
                    continue
                if not isinstance(d, dict) or "metric" not in d or "value" not in d:
                    continue
                cfg = d.get("config") or {}
                rl = d.get("roofline") or {}
                nv = d.get("roofline_nvlink") or {}
                op = d.get("owner_phase") or {}
                e2e = d.get("e2e") or {}
                ck = d.get("clocks") or {}
                yield {
                    "file": os.path.relpath(f), "impl": d.get("impl", "ours"),
                    "workload": cfg.get("workload", cfg.get("model", "")),
                    "n_gpus": d.get("n_gpus"), "workers": cfg.get("workers"),
                    "chunk_bytes": cfg.get("chunk_bytes"),
                    "mode": (cfg.get("mode") or "")[:60], "kernel": cfg.get("kernel", ""),
                    "value_GBps": d.get("value"), "ms_per_step": d.get("ms_per_step"),
                    "exchanges_per_s": d.get("exchanges_per_s"), "scaling": d.get("scaling"),
                    "roofline_bound": rl.get("bound"), "roofline_achieved": rl.get("achieved"),
                    "roofline_peak": rl.get("peak"), "roofline_frac": rl.get("frac"),
                    "nvlink_frac": nv.get("frac"), "owner_phase_GBps": op.get("value"),
                    "e2e_GBps": e2e.get("value"), "sm_mhz": ck.get("sm_mhz"),
                    "throttle_reasons": ";".join(ck.get("reasons") or []),
                }


def main(argv):
    w = csv.DictWriter(sys.stdout, fieldnames=COLUMNS, lineterminator="\n")
    w.writeheader()
    for r in rows(argv or ["profiles"]):
        w.writerow(r)


if __name__ == "__main__":
    main(sys.argv[1:])
