#!/usr/bin/env python3
"""Benchmark of the PHub hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config vgg19]
    torchrun --nproc-per-node N bench.py --gpus N ...      (driver, N > 1)
    python bench.py --impl reference ...                    (CPU oracle arm)

One step = one full parameter-exchange round of the 8-worker job: every
worker's push, the fused tall aggregation + Nesterov update of every chunk,
and the pull.  N = 1: all 8 workers' gradients are resident in HBM and pushed
zero-copy (mode M1).  N > 1: one process per GPU, 8/N workers per
GPU, chunks sharded by owner (mode M3); `--mode auto` runs the scheduled
exchange (one launch per GPU, each owner range moved partly as
raw worker slices and partly as a rank-by-rank worker-order chain, mixed so
the busiest NVLink port moves the fewest bytes -- the chain at N = 2, the push
exchange at N = 8, a mix in between); the block-streamed chain (chain), the
all-store push exchange (push), the owner-sharded peer-load kernel (p2p),
NCCL send/recv and an NCCL all-reduce baseline are options.
Total work is fixed as N grows ("scaling": "strong").  `--mode hier` is the
hierarchical reduction (one 8-worker rack per GPU, weak scaling, NEXT-4).

metric: aggregated gradient GB/s = 8 * 4E / t_step (plus exchanges/s = 8 / t_step).
Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import datetime
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "aggregated gradient GB/s + model exchanges/sec (8 workers) at 1/2/4/8 B200"
PAPER_GBS = 41.4   # 72.08 exchanges/s x 574.7 MB (VGG-19, 8 workers, PBox)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="vgg19")
    ap.add_argument("--workers", type=int, default=None)
    ap.add_argument("--chunk-bytes", type=int, default=None)
    ap.add_argument("--kernel", default="auto", choices=["auto", "flat", "flat128", "tiles", "wide", "bulk"])
    ap.add_argument("--cache", default="resident", choices=["enabled", "bypass", "resident"],
                    help="L2 policy: resident = a fixed 32 MiB slice of w stays in L2 across "
                         "rounds, the rest evict-first (default, measured fastest); bypass = "
                         "every stream evict-first; enabled = all of w' evict-last (P:911)")
    ap.add_argument("--resident-mb", type=int, default=-1,
                    help="resident policy: MiB of w kept in L2 across rounds (-1: library default)")
    ap.add_argument("--e2e-steps", type=int, default=16,
                    help="e2e rounds timed (the pipeline's fill + drain is amortised over them)")
    ap.add_argument("--e2e-streams", type=int, default=1,
                    help="copy streams per direction in the 1-GPU e2e measurement")
    ap.add_argument("--grid", type=int, default=0, help="CTAs for the flat kernel (0 = auto)")
    ap.add_argument("--tile-elems", type=int, default=0, help="chunk-tile kernel tile size")
    ap.add_argument("--oneshot", type=int, default=-1, help="flat kernel one-vector-per-thread grid")
    ap.add_argument("--graph", action="store_true",
                    help="also time the round replayed from a captured CUDA graph")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-rounds", type=int, default=3,
                    help="full-model oracle rounds per thread count (median reported)")
    ap.add_argument("--cache-table", action="store_true",
                    help="N=1: also time the caching table of P:913-935 on B200 (fused kernel "
                         "with w' evict-last vs all evict-first, alone and followed by the pull)")
    ap.add_argument("--owner-policy", default="contig", choices=["contig"])
    ap.add_argument("--pieces", type=int, default=8, help="chain mode pipeline pieces")
    ap.add_argument("--chain-sync", default="blocks", choices=["blocks", "flags", "barrier"])
    ap.add_argument("--chain-block", type=int, default=0,
                    help="chain mode: elements per block flag (sync=blocks; 0 = by model size)")
    ap.add_argument("--hier-block", type=int, default=32768,
                    help="hier mode: elements per block flag")
    ap.add_argument("--push-block", type=int, default=12288,
                    help="push mode: elements per block flag")
    ap.add_argument("--sched-block", type=int, default=0,
                    help="sched mode: elements per item block (0: 16384 at G = 2, else 12288)")
    ap.add_argument("--sched-lag", type=int, default=-1,
                    help="sched mode: blocks of progress each chain stage / consumer lags "
                         "(-1: 0 at G = 2, else 64)")
    ap.add_argument("--sched-taper", type=int, default=-1,
                    help="sched mode: blocks at each part's ends cut 4x finer (-1: 0 at G = 2, "
                         "else 8)")
    ap.add_argument("--sched-host-barrier", action="store_true",
                    help="sched mode: NCCL start/end barriers instead of the in-kernel ones")
    ap.add_argument("--sched-consumers", type=int, default=0,
                    help="sched mode: CTAs serving the consumer lane (0 = auto)")
    ap.add_argument("--sched-weights", default="",
                    help="sched mode: comma-separated owner shares (default: sharded.SCHED_TABLE)")
    ap.add_argument("--sched-raw", default="",
                    help="sched mode: comma-separated RAW fraction per owner (with --sched-weights)")
    ap.add_argument("--chain-producer-grid", type=int, default=0,
                    help="chain mode: CTAs of the partial-sum launch on non-last ranks")
    ap.add_argument("--chain-consumer-grid", type=int, default=0,
                    help="chain mode: CTAs of the fused launch on the last rank")
    ap.add_argument("--mode", default="auto",
                    choices=["auto", "p2p", "push", "sched", "chain", "nccl", "allreduce", "hier"],
                    help="N>1 exchange of the 8-worker job: chained (chain), owner-sharded "
                         "all-store (push) or peer-load (p2p) kernels, NCCL send/recv (nccl), "
                         "NCCL all-reduce baseline (allreduce); hier: hierarchical reduction, "
                         "one 8-worker rack per GPU (SURVEY NEXT-4, weak scaling)")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi style clock/throttle sampling through NVML during the timed region."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x1: "gpu_idle"}

    def __init__(self, device_index: int, period: float = 0.01):
        self.samples, self.reasons = [], set()
        self.ok = False
        self.period = period
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = self._handle(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _handle(self, idx):
        import torch
        try:
            uuid = str(torch.cuda.get_device_properties(idx).uuid)
            return self.nv.nvmlDeviceGetHandleByUUID(("GPU-" + uuid).encode()
                                                     if not uuid.startswith("GPU-") else uuid.encode())
        except Exception:
            return self.nv.nvmlDeviceGetHandleByIndex(idx)

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append(mhz)
                for bit, name in self.REASONS.items():
                    if r & bit and bit not in (0x1,):
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(self.period)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if self.ok:
            self._stop.set()
            self.t.join()
            # one final sample so even a very short region has a reading
            if not self.samples:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def hbm_copy_probe(dev, reps=10):
    """Same-run HBM probe, MEASURED_PEAKS' recipe: b.copy_(a) over 1 Gi bf16
    elements, read + write bytes, best of `reps` (CUDA events)."""
    import torch
    a = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev)
    b = torch.empty_like(a)
    best = float("inf")
    for _ in range(reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    del a, b
    torch.cuda.empty_cache()
    return round(2 * 2 * (1 << 30) / best / 1e9, 1)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(config, kernel):
    """(dram bytes per launch, source) of the hot kernel from the committed ncu
    summary -- an `ncu --set full` capture of an earlier run, NOT measured in
    this run (ncu cannot run inside a timed bench)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as f:
        d = json.load(f)
    ent = d.get(f"{config}:{kernel}") or d.get(config)
    if not ent:
        return None, None
    return ent.get("dram_bytes_per_launch"), (
        f"committed ncu --set full capture ({ent.get('source', 'profiles/ncu_traffic.json')}), "
        "dram__bytes_read.sum + dram__bytes_write.sum per launch; not measured in this run")


# -------------------------------------------------------------- CPU oracle
_CPU_INPUTS = {}


def cpu_inputs(config_name, workers):
    """Host arrays of the FULL workload: the same counter-based streams the GPU
    arm generates (workloads.generate; torch CPU ops, all host threads)."""
    import torch
    from workloads import grad_stream, manifest
    from workloads.generate import values_torch
    key = (config_name, workers)
    if key not in _CPU_INPUTS:
        _CPU_INPUTS.clear()
        sizes = manifest(config_name)
        E = sum(sizes)
        torch.set_num_threads(len(os.sched_getaffinity(0)))
        grads = [values_torch(grad_stream(w), 0, E, 25, "cpu").numpy() for w in range(workers)]
        _CPU_INPUTS[key] = (sizes, grads, values_torch(1, 0, E, 20, "cpu").numpy(),
                            values_torch(2, 0, E, 25, "cpu").numpy())
    return _CPU_INPUTS[key]


def host_cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return ""


def cpu_oracle_rounds(config_name, workers, chunk_bytes, rounds, nthreads=None):
    """The CPU oracle, as it stands, on `rounds` FULL rounds of the workload
    (every key, every worker, no sampling); returns the per-round seconds."""
    import oracle
    sizes, grads, w0, v0 = cpu_inputs(config_name, workers)
    nt = nthreads or len(os.sched_getaffinity(0))
    times = []
    for _ in range(rounds):
        t0 = time.perf_counter()
        oracle.round_(sizes, grads, w0, v0, 0.1, 0.9, chunk_bytes=chunk_bytes, keep_agg=False,
                      nthreads=nt)
        times.append(time.perf_counter() - t0)
    return times, nt


def cpu_baseline(config_name, workers, chunk_bytes, rounds):
    """SURVEY 8(d) "Oracle timing": median of `rounds` full rounds on all host
    cores (OpenMP static over vkeys: PHub's chunk -> core layout), and
    the same on one thread."""
    from workloads import manifest
    E = sum(manifest(config_name))
    t_all, nt = cpu_oracle_rounds(config_name, workers, chunk_bytes, rounds)
    t_one, _ = cpu_oracle_rounds(config_name, workers, chunk_bytes, rounds, nthreads=1)
    m_all, m_one = statistics.median(t_all), statistics.median(t_one)
    return {"value": round(workers * 4 * E / m_all / 1e9, 3), "unit": "GB/s", "cores": nt,
            "kind": "oracle",
            "sample": f"full {config_name} round ({E} elements x {workers} workers, every key, no "
                      f"sampling), {chunk_bytes} B chunks, OpenMP static over vkeys ({nt} threads, "
                      f"PHub chunk->core layout); median of {len(t_all)} rounds",
            "ms_per_round": round(m_all * 1e3, 2), "exchanges_per_s": round(workers / m_all, 3),
            "host_cpu": host_cpu_model(), "host_cores_available": len(os.sched_getaffinity(0)),
            "single_thread": {"value": round(workers * 4 * E / m_one / 1e9, 3), "unit": "GB/s",
                              "cores": 1, "ms_per_round": round(m_one * 1e3, 2),
                              "rounds": len(t_one)}}


def run_reference(args):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only); every
    warm-up and timed step is one FULL round of the workload on all host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from workloads.manifests import CONFIGS
    from workloads import manifest
    mname, N, cb = CONFIGS[args.config]
    N = args.workers or N
    cb = args.chunk_bytes or cb
    E = sum(manifest(mname))
    cpu_oracle_rounds(mname, N, cb, args.warmup)
    times, nt = cpu_oracle_rounds(mname, N, cb, args.steps)
    t_round = statistics.median(times)
    value = N * 4 * E / t_round / 1e9
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t_round * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": round(value / PAPER_GBS, 4), "dtype": "f32",
        "data": "synthetic", "exchanges_per_s": round(N / t_round, 3),
        "config": {"workload": args.config, "keys": len(manifest(mname)), "E": E, "workers": N,
                   "chunk_bytes": cb, "timing": "median over the timed steps; one step = one "
                                                 "full round (no sampling, no extrapolation)"},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": nt, "kind": "oracle",
                         "sample": f"full {mname} round every step ({E} elements x {N} workers)",
                         "host_cpu": host_cpu_model()},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))


def pcie_probe(dev, mib=1024, reps=5, h_in=None, h_out=None):
    """Same-run PCIe ceiling for the e2e numbers: pinned host <-> device copies
    of `mib` MiB (H2D alone, D2H alone, both at once on two streams), best of
    `reps` (CUDA events).  h_in / h_out: the e2e run's own pinned buffers (the
    same host pages, hence the same NUMA placement, as the measurement it is
    held against -- fresh allocations can land elsewhere and measure lower)."""
    import torch
    n = mib * (1 << 20) // 4
    h_in = h_in[:n] if h_in is not None else torch.ones(n, pin_memory=True)
    h_out = h_out[:n] if h_out is not None else torch.empty(n, pin_memory=True)
    n = min(h_in.numel(), h_out.numel())
    d_in = torch.empty(n, device=dev)
    d_out = torch.ones(n, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    cur = torch.cuda.current_stream(dev)

    def timed(fn):
        best = float("inf")
        for _ in range(reps + 1):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            a.record(cur)
            fn()
            b.record(cur)
            torch.cuda.synchronize(dev)
            best = min(best, a.elapsed_time(b) / 1e3)
        return best

    def both():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    th = timed(lambda: d_in.copy_(h_in, non_blocking=True))
    td = timed(lambda: h_out.copy_(d_out, non_blocking=True))
    tb = timed(both)
    nb = 4 * n
    out = {"h2d_gbs": round(nb / th / 1e9, 2), "d2h_gbs": round(nb / td / 1e9, 2),
           "bidir_gbs_per_direction": round(nb / tb / 1e9, 2), "bytes": nb,
           "how": f"pinned {nb / 2**20:.0f} MiB copies, best of {reps}, CUDA events"}
    del h_in, h_out, d_in, d_out
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------ ours
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    from workloads.manifests import CONFIGS
    mname, N, cb = CONFIGS[args.config]
    N = args.workers or N
    cb = args.chunk_bytes or cb
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 or world > 1 or args.mode == "hier":
        if world == 1:           # single-process hier (one rack): a 1-rank process group
            import socket
            with socket.socket() as s_:
                s_.bind(("127.0.0.1", 0))
                port = s_.getsockname()[1]
            for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", str(port)),
                         ("RANK", "0"), ("WORLD_SIZE", "1"), ("LOCAL_RANK", "0")):
                os.environ.setdefault(k, v)
        return bench_multi(args, mname, N, cb)
    return bench_single(args, mname, N, cb)


NVLINK_PEER_GBS = 770.0   # B200_PROFILING.md: measured peer copy per direction per GPU


def nccl_allgather_busbw(dev, G, mib=256, reps=5):
    """Same-run NVLink probe: NCCL all-gather of `mib` MiB per
    rank, bus bandwidth = (G-1)/G * total bytes / t (nccl-tests' definition),
    best of `reps`, max time over ranks."""
    import torch
    import torch.distributed as dist
    n = mib * (1 << 20) // 4
    src = torch.ones(n, dtype=torch.float32, device=dev)
    dst = torch.empty(n * G, dtype=torch.float32, device=dev)
    best = float("inf")
    for _ in range(reps + 2):
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dist.all_gather_into_tensor(dst, src)
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / 1e3], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        best = min(best, float(t.item()))
    del src, dst
    torch.cuda.empty_cache()
    return round((G - 1) / G * 4 * n * G / best / 1e9, 1)


def hier_model(P, R, b_nvlink, b_hbm):
    """The paper's benefit model for hierarchical reduction (P:760-763,
    phub_hier_beneficial) evaluated with this box's measured rates: a rack's
    PBox is a GPU whose network port is its NVLink (B_PBox = same-run NCCL
    all-gather bus bandwidth), its P workers' gradients stream from its HBM
    (B_Wkr = measured HBM copy rate / P), and the NVSwitch core is
    non-blocking (B_Core = R x B_PBox).  Reported next to the measured rounds;
    DESIGN.md R18 discusses the mapping."""
    from paper_1805_07891_b200 import capi
    bw = {"b_pbox": float(b_nvlink), "b_wkr": float(b_hbm) / P, "b_core": R * float(b_nvlink)}
    out = {"workers_per_rack": P, "racks": R, **{k: round(v, 1) for k, v in bw.items()},
           "unit": "GB/s"}
    for mode, name in ((capi.PHUB_CROSS_RACK_SHARDED, "sharded"),
                       (capi.PHUB_CROSS_RACK_RING, "ring")):
        ben, lhs, rhs = capi.phub_hier_beneficial(P, R, bw["b_pbox"], bw["b_wkr"], bw["b_core"],
                                                  mode)
        out[name] = {"beneficial": ben, "lhs": lhs, "rhs": rhs}
    return out


def owner_phase_ms(sizes, N, cb, rank, G, steps, warmup, dev):
    """Mode M2: this rank's owner kernel alone, with the N workers'
    slices of its owned range already resident in its HBM (PHub's pushes land
    by DMA at the owner).  Returns the mean kernel ms (CUDA
    events on the launching stream)."""
    import torch
    from paper_1805_07891_b200 import PHub, capi
    from workloads import grad_stream
    from workloads.generate import values_torch
    hub = PHub(sizes, N, chunk_size_bytes=cb, device=dev.index, num_owners=G, owner_rank=rank,
               owner_policy="contig")
    b, e = hub.owner_range()
    bufs = [values_torch(grad_stream(w), b, e - b, 25, dev) for w in range(N)]
    stream = torch.cuda.current_stream(dev)

    def one():
        for w in range(N):
            hub.push(w, bufs[w], key=capi.PHUB_OWNED_RANGE)
        hub.aggregate_optimize()

    for _ in range(warmup):
        one()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    t0.record(stream)
    for _ in range(steps):
        one()
    t1.record(stream)
    torch.cuda.synchronize(dev)
    ms = t0.elapsed_time(t1) / steps
    owned = hub.owned_elements()
    hub.close()
    del bufs
    return ms, owned


def bench_multi(args, mname, N, cb):
    """M3: 8 workers hosted N/G per GPU, chunks sharded by owner.
    mode p2p : one fused kernel per owner reads peers' gradients and writes peers'
               replicas over NVLink (stream-ordered NCCL barrier before/after);
    mode nccl: NCCL grouped send/recv push, fused kernel, NCCL all-gather-v pull."""
    import torch
    import torch.distributed as dist
    from paper_1805_07891_b200.sharded import (AllReduceBaseline, ChainShardedPHub, HierPHub,
                                               P2PShardedPHub, PushShardedPHub, SchedShardedPHub,
                                               ShardedPHub)
    from workloads import grad_stream, manifest
    from workloads.generate import values_torch

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=300))
    rank, G = dist.get_rank(), dist.get_world_size()
    sizes = manifest(mname)
    if args.mode == "auto":      # the scheduled exchange: byte-balanced ports at every G (8.6)
        args.mode = "sched"
    hier = args.mode == "hier"
    push = args.mode == "push"
    sched = args.mode == "sched"
    chain = args.mode in ("chain", "hier", "push", "sched")   # the round is one exchange() call
    p2p = args.mode in ("p2p", "chain", "hier", "push", "sched")
    ar = args.mode == "allreduce"
    NT = N * G if hier else N                   # workers in the job
    try:
        if hier:
            sh = HierPHub(sizes, workers_per_rack=N, chunk_size_bytes=cb, device=local,
                          block=args.hier_block)
        elif push:
            sh = PushShardedPHub(sizes, N, chunk_size_bytes=cb, device=local,
                                 block=args.push_block)
        elif sched:
            fl = lambda x: [float(v) for v in x.split(",")] if x else None  # noqa: E731
            sh = SchedShardedPHub(sizes, N, chunk_size_bytes=cb, device=local,
                                  block=args.sched_block, lag=args.sched_lag,
                                  consumer_ctas=args.sched_consumers, taper=args.sched_taper,
                                  device_barrier=not args.sched_host_barrier,
                                  weights=fl(args.sched_weights), raw_frac=fl(args.sched_raw))
        elif chain:
            sh = ChainShardedPHub(sizes, N, chunk_size_bytes=cb, device=local, pieces=args.pieces,
                                  sync=args.chain_sync, block=args.chain_block)
            from paper_1805_07891_b200 import capi as _c
            if args.chain_producer_grid and not sh.last:
                sh.hub.set_option(_c.PHUB_OPT_GRID, args.chain_producer_grid)
            if args.chain_consumer_grid and sh.last:
                sh.hub.set_option(_c.PHUB_OPT_GRID, args.chain_consumer_grid)
        else:
            cls = {"p2p": P2PShardedPHub, "nccl": ShardedPHub,
                   "allreduce": AllReduceBaseline}[args.mode]
            sh = cls(sizes, N, chunk_size_bytes=cb, device=local)
    except Exception as e:  # noqa: BLE001 -- every rank raises together (see sharded.py)
        if not p2p:
            raise
        print(f"[bench] p2p exchange unavailable ({e}); using the NCCL exchange", file=sys.stderr)
        args.mode, p2p, chain = "nccl", False, False
        sh = ShardedPHub(sizes, N, chunk_size_bytes=cb, device=local)
    hub, plan = sh.hub, getattr(sh, "plan", None)
    from paper_1805_07891_b200 import capi
    if args.grid:
        hub.set_option(capi.PHUB_OPT_GRID, args.grid)
    if args.oneshot >= 0:
        hub.set_option(capi.PHUB_OPT_FLAT_ONESHOT, args.oneshot)
    if args.tile_elems:
        hub.set_option(capi.PHUB_OPT_TILE_ELEMS, args.tile_elems)
    if args.kernel != "auto":
        hub.set_option(capi.PHUB_OPT_KERNEL, {"flat": capi.PHUB_KERNEL_FLAT,
                                              "flat128": capi.PHUB_KERNEL_FLAT128,
                                              "tiles": capi.PHUB_KERNEL_TILES,
                                              "wide": capi.PHUB_KERNEL_WIDE,
                                              "bulk": capi.PHUB_KERNEL_BULK}[args.kernel])
    E, Ep = hub.E, hub.E_padded
    idx = torch.as_tensor(hub.padded_index(), device=dev)
    hub.load_state(values_torch(1, 0, E, 20, dev), values_torch(2, 0, E, 25, dev))
    grads = sh.gradients() if p2p else {}
    for w in sh.hosted:
        b = grads[w] if p2p else torch.zeros(Ep, dtype=torch.float32, device=dev)
        b[idx] = values_torch(grad_stream(rank * N + w if hier else w), 0, E, 25, dev)
        grads[w] = b
    del idx
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)

    def one(i=None):
        if chain:                      # the whole round is phases of fused kernels + barriers
            if i is not None:
                ev[i][0].record(stream)
            sh.exchange()
            if i is not None:
                ev[i][1].record(stream)
            return
        if ar:
            hosted = sh.hosted
            sh.sum.copy_(grads[hosted[0]])
            for w in hosted[1:]:
                sh.sum.add_(grads[w])
            dist.all_reduce(sh.sum)
            hub.push(0, sh.sum)
        elif p2p:
            sh.barrier()
            sh.push()
        else:
            sh.push(grads)
        if i is not None:
            ev[i][0].record(stream)
        hub.aggregate_optimize()
        if i is not None:
            ev[i][1].record(stream)
        if p2p:
            sh.barrier()
        elif not ar:
            sh.pull()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for _ in range(args.warmup):
        one()
    torch.cuda.synchronize()
    dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    k0 = hub.kernel_launches
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    dist.barrier()
    t0.record(stream)
    for i in range(args.steps):
        one(i)
    t1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clocks.stop()
    launches = hub.kernel_launches - k0
    if chain:
        sh.check()               # collective: raises on every rank if any device wait expired
    mine = {"rank": rank, "ms": t0.elapsed_time(t1) / args.steps,
            "k_ms": sum(a.elapsed_time(b) for a, b in ev) / args.steps,
            "owned": hub.owned_elements(), "launches": launches, "clocks": clocks.summary()}
    if plan is not None:
        mine["out"], mine["in"] = plan.nvlink_bytes_out(), plan.nvlink_bytes_in()
    if hier:    # rack aggregate of every other owner's range out, w' of the own range to G-1
        from paper_1805_07891_b200.sharded import hier_nvlink_bytes
        mine["out"], mine["in"] = hier_nvlink_bytes(
            [hub.owner_range(o) for o in range(G)], Ep, rank)
    elif push:   # same bytes as the owner-sharded P2P exchange (plan), all as stores
        pass
    elif sched:  # RAW slices + CHAIN partials + final sums + replica stores (byte model)
        mine["out"], mine["in"] = sh.nvlink_bytes()
    elif chain:  # one partial per link per round; the last rank stores w' into G-1 replicas
        from paper_1805_07891_b200.sharded import chain_nvlink_bytes
        mine["out"], mine["in"] = chain_nvlink_bytes(Ep, G, rank)
    if p2p:     # M2: the owner kernel alone on resident slices (NCCL mode: its k_ms already is)
        mine["m2_ms"], mine["m2_owned"] = owner_phase_ms(sizes, NT, cb, rank, G, args.steps,
                                                         args.warmup, dev)
    else:
        mine["m2_ms"], mine["m2_owned"] = mine["k_ms"], mine["owned"]
    allr = [None] * G
    dist.all_gather_object(allr, mine)
    ag_busbw = nccl_allgather_busbw(dev, G) if G > 1 else None

    e2e = None
    if not args.no_e2e and not ar:
        host_g = {w: torch.empty(Ep, dtype=torch.float32, pin_memory=True) for w in sh.hosted}
        for w in sh.hosted:
            host_g[w].copy_(grads[w])
        host_o = {w: torch.empty(Ep, dtype=torch.float32, pin_memory=True) for w in sh.hosted}

        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        total = args.e2e_steps + 1
        ev_x = [torch.cuda.Event() for _ in range(total)]
        ev_in = [torch.cuda.Event() for _ in range(total)]
        ev_out = [torch.cuda.Event() for _ in range(total)]

        def e2e_round(k):
            """fused modes: H2D of round k (slot k % 2) on s_in overlaps the D2H of
            round k-1 on s_out; the exchange waits for both."""
            if not p2p:
                sh.exchange_host(host_g, grads, host_o)
                return
            slot = k % 2
            if k >= 2:
                s_in.wait_event(ev_x[k - 2])            # slot free: exchange k-2 is done
            g = sh.gradients(slot)
            with torch.cuda.stream(s_in):
                for w in sh.hosted:
                    g[w].copy_(host_g[w], non_blocking=True)
            ev_in[k].record(s_in)
            stream.wait_event(ev_in[k])
            if k >= 1:                                  # the pulls that read the replica
                stream.wait_event(ev_out[k - 1])        # this round overwrites
            sh.exchange(slot)
            ev_x[k].record(stream)
            s_out.wait_event(ev_x[k])
            with torch.cuda.stream(s_out):
                for w in sh.hosted:
                    host_o[w].copy_(sh.replica, non_blocking=True)
            ev_out[k].record(s_out)

        e2e_round(0)
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        s_in.wait_event(a)
        s_out.wait_event(a)
        for k in range(1, total):
            e2e_round(k)
        if p2p:
            stream.wait_event(ev_out[total - 1])
        b.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / args.e2e_steps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        te = float(t.item()) / 1e3
        if chain:
            sh.check()
        w0 = sh.hosted[0]
        probe = pcie_probe(dev, h_in=host_g[w0], h_out=host_o[w0])
        del host_g, host_o
        pr = [None] * G
        dist.all_gather_object(pr, probe)
        slowest = min(pr, key=lambda x: x["bidir_gbs_per_direction"])
        per_gpu_dir = len(sh.hosted) * 4 * Ep / te / 1e9
        e2e = {"value": round(NT * 4 * E / te / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": NT * 4 * Ep, "d2h_bytes_per_step": NT * 4 * Ep,
               "steps": args.e2e_steps, "ms_per_step": round(te * 1e3, 3),
               "pcie_probe_slowest_rank": slowest,
               "gbs_per_direction_per_gpu": round(per_gpu_dir, 2),
               "frac_of_pcie_bidir": round(per_gpu_dir / slowest["bidir_gbs_per_direction"], 4),
               "path": f"{type(sh).__name__}: H2D of hosted grads -> exchange ({args.mode}) -> "
                       f"D2H of the replica per hosted worker" +
                       (" ; rounds pipelined (2 gradient slots, H2D of k+1 || D2H of k)"
                        if p2p else "")}
    if rank == 0:
        ms_step = max(r["ms"] for r in allr)
        k_ms = max(r["k_ms"] for r in allr)
        t_step = ms_step / 1e3
        value = NT * 4 * E / t_step / 1e9
        slow = max(allr, key=lambda r: r["k_ms"])
        m2_slow = max(allr, key=lambda r: r["m2_ms"])
        m2_ms = m2_slow["m2_ms"]
        achieved = (4 * NT + 16) * slow["owned"] / (slow["k_ms"] / 1e3) / 1e9
        peak, peak_src = measured_peaks()
        nv_bytes = max(max(r["out"], r["in"]) for r in allr) if not ar else \
            int(2 * (G - 1) / G * 4 * Ep)              # ring all-reduce bytes per direction
        nv_ach = nv_bytes / t_step / 1e9
        reasons = sorted(set(x for r in allr for x in r["clocks"].get("reasons", [])))
        sm = [r["clocks"]["sm_mhz"] for r in allr if r["clocks"].get("sm_mhz")]
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": G,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak" if hier else "strong",
            "vs_baseline": None if hier else round(value / PAPER_GBS, 2), "dtype": "f32",
            "data": "synthetic", "exchanges_per_s": round(NT / t_step, 1),
            "config": {"workload": args.config, "keys": len(sizes), "E": E, "E_padded": Ep,
                       "workers": NT, "workers_per_gpu": NT // G, "chunk_bytes": cb,
                       "mode": (f"NEXT-4 hierarchical reduction (P:746-763): one rack of {N} "
                                f"workers per GPU ({NT} in all), rack aggregate -> cross-rack "
                                f"aggregation in rack order over NVLink -> Nesterov on owner "
                                f"ranges + w' into every rack's replica; one launch per GPU, "
                                f"{args.hier_block}-element blocks") if hier else
                               ("M3 (full exchange) push: one ticket-ordered launch per GPU "
                                "stores its workers' raw slices into every other owner's inbox "
                                "over NVLink and sums its own range over all workers in worker "
                                "order -> Nesterov -> w' into every replica (all NVLink traffic "
                                "as stores)") if push else
                               (f"M3 (full exchange) sched: one ticket-ordered launch per GPU "
                                f"executes its item program -- per owner range a RAW part "
                                f"(raw worker slices stored into the owner) and a CHAIN part "
                                f"(rank-by-rank worker-order partials, finished sum stored into "
                                f"the owner), mixed per owner so the busiest NVLink port moves "
                                f"the fewest bytes; owner shares {[round(x, 4) for x in sh.shares]}"
                                f", RAW fractions {[round(x, 4) for x in sh.raw_frac]}, "
                                f"{sh.block}-element blocks, lag {sh.lag}, taper {sh.taper}, "
                                f"consumer-lane CTAs {args.sched_consumers or 'auto'}, "
                                f"{'NCCL' if args.sched_host_barrier else 'in-kernel'} round "
                                f"barriers")
                               if sched else
                               (f"M3 (full exchange) chain: rank-ordered partial sums over "
                                f"NVLink, last rank fused Nesterov + replica stores, " +
                                (f"one launch per rank streamed by per-block device flags "
                                 f"({sh.block} elements/block, partial stored into the next "
                                 f"rank's inbox)"
                                 if args.chain_sync == "blocks" else
                                 f"pipelined over {args.pieces} pieces ({args.chain_sync} sync)"))
                               if chain else
                               ("M3 (full exchange) p2p: one fused kernel per owner reads peer "
                                "gradients + writes peer replicas over NVLink, NCCL barrier "
                                "before/after") if p2p else
                               ("BASELINE (not exact, NEXT-3): local torch sum of hosted workers, "
                                "NCCL all-reduce, libphub NAG on the whole model on every GPU")
                               if ar else
                               ("M3 (full exchange) nccl: NCCL grouped send/recv push, fused "
                                "kernel on owner range, NCCL all-gather-v pull"),
                       "parallelism": f"owner-sharded x{G}", "kernel": args.kernel,
                       "grid": args.grid,
                       "l2": "no flush: inputs exceed L2"},
            "owner_phase": None if ar else {
                "mode": "M2 (SURVEY 8(d)): owner kernel alone, the N workers' slices of its "
                        "range resident in its HBM (pushes landed by DMA, P:895/P:933); "
                        "max over ranks; NOT the headline (no NVLink transfer)",
                "kernel_ms": round(m2_ms, 4),
                "value": round(NT * 4 * E / (m2_ms / 1e3) / 1e9, 1), "unit": "GB/s",
                "hbm_frac": round((4 * NT + 16) * m2_slow["m2_owned"] / (m2_ms / 1e3) / 1e9 /
                                  measured_peaks()[0], 4)},
            "roofline": ({"bound": "nvlink", "achieved": round(nv_bytes / (k_ms / 1e3) / 1e9, 1),
                          "peak": NVLINK_PEER_GBS, "unit": "GB/s",
                          "frac": round(nv_bytes / (k_ms / 1e3) / 1e9 / NVLINK_PEER_GBS, 4),
                          "traffic": None,
                          "kernel": ("hierarchical exchange round (k_hier, incl. the "
                                     "end barrier)") if hier else
                                    ("push exchange round (k_hier worker-order, incl. the end "
                                     "barrier)") if push else
                                    ("scheduled exchange round (k_sched, incl. the end "
                                     "barrier)") if sched else
                                    ("chained exchange round (partial-sum + fused kernels, "
                                     "incl. barriers)") if chain else
                                    ("fused exchange kernel (k_flat with peer loads/stores), "
                                     "slowest owner"), "kernel_ms": round(k_ms, 4),
                          "bytes_per_launch_max_dir": nv_bytes,
                          "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per "
                                         "direction"} if p2p else
                         {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                          "unit": "GB/s", "frac": round(achieved / peak, 4),
                          "traffic": ncu_traffic(args.config, "flat")[0],
                          "traffic_source": ncu_traffic(args.config, "flat")[1],
                          "kernel": "phub_agg_nag (k_flat) on the slowest owner",
                          "kernel_ms": round(slow["k_ms"], 4), "peak_source": peak_src}),
            "roofline_nvlink": {"bound": "nvlink", "achieved": round(nv_ach, 1),
                                "peak": NVLINK_PEER_GBS, "unit": "GB/s",
                                "frac": round(nv_ach / NVLINK_PEER_GBS, 4),
                                "bytes_per_step_max_dir": nv_bytes,
                                "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s "
                                               "per direction (900 nominal)",
                                "same_run_nccl_allgather_busbw": ag_busbw,
                                "frac_of_nccl_allgather": round(nv_ach / ag_busbw, 4)
                                if ag_busbw else None},
            "clocks": {"sm_mhz": statistics.median(sm) if sm else None,
                       "sm_max_mhz": allr[0]["clocks"].get("sm_max_mhz"), "reasons": reasons},
            "gpu_launches": sum(r["launches"] for r in allr),
            "hier_model": hier_model(N, G, ag_busbw, measured_peaks()[0])
            if hier and G > 1 and ag_busbw else None,
            "e2e": e2e,
            "cpu_baseline": None,
        }
        print(json.dumps(out))
    sh.close()
    dist.barrier()
    dist.destroy_process_group()


def bench_single(args, mname, N, cb):
    import torch
    from paper_1805_07891_b200 import PHub, capi
    from workloads import grad_stream, manifest
    from workloads.generate import values_torch

    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    sizes = manifest(mname)
    hub = PHub(sizes, N, chunk_size_bytes=cb, device=0)
    kern = {"auto": capi.PHUB_KERNEL_AUTO, "flat": capi.PHUB_KERNEL_FLAT,
            "flat128": capi.PHUB_KERNEL_FLAT128, "tiles": capi.PHUB_KERNEL_TILES,
            "wide": capi.PHUB_KERNEL_WIDE, "bulk": capi.PHUB_KERNEL_BULK}[args.kernel]
    if kern == capi.PHUB_KERNEL_WIDE:
        hub.close()
        hub = PHub(sizes, N, chunk_size_bytes=cb, device=0, keep_aggregate=True)
    hub.set_option(capi.PHUB_OPT_KERNEL, kern)
    hub.set_option(capi.PHUB_OPT_CACHE, {"bypass": capi.PHUB_CACHE_BYPASS,
                                         "enabled": capi.PHUB_CACHE_ENABLED,
                                         "resident": capi.PHUB_CACHE_RESIDENT}[args.cache])
    if args.resident_mb >= 0:
        hub.set_option(capi.PHUB_OPT_L2_RESIDENT, args.resident_mb << 20)
    if args.grid:
        hub.set_option(capi.PHUB_OPT_GRID, args.grid)
    if args.tile_elems:
        hub.set_option(capi.PHUB_OPT_TILE_ELEMS, args.tile_elems)
    if args.oneshot >= 0:
        hub.set_option(capi.PHUB_OPT_FLAT_ONESHOT, args.oneshot)
    E, Ep = hub.E, hub.E_padded
    idx = torch.as_tensor(hub.padded_index(), device=dev)
    hub.load_state(values_torch(1, 0, E, 20, dev), values_torch(2, 0, E, 25, dev))
    grads = []
    for w in range(N):
        b = torch.zeros(Ep, dtype=torch.float32, device=dev)
        b[idx] = values_torch(grad_stream(w), 0, E, 25, dev)
        grads.append(b)
    del idx
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)

    batch = [(w, capi.PHUB_ALL_KEYS, grads[w]) for w in range(N)]

    def step():
        hub.push_batch(batch)                 # N zero-copy BORROW pushes: host bookkeeping only
        hub.aggregate_optimize()              # one fused kernel on `stream`

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    clocks.start()
    k0 = hub.kernel_launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t_start.record(stream)
    for i in range(args.steps):
        hub.push_batch(batch)
        ev[i][0].record(stream)
        hub.aggregate_optimize()
        ev[i][1].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    clocks.stop()
    launches = hub.kernel_launches - k0
    ms_step = t_start.elapsed_time(t_end) / args.steps
    k_ms = [a.elapsed_time(b) for a, b in ev]
    k_ms_mean = sum(k_ms) / len(k_ms)
    t_step = ms_step / 1e3
    value = N * 4 * E / t_step / 1e9
    owned = hub.owned_elements()
    algo_bytes = (4 * N + 16) * owned
    achieved = algo_bytes / (k_ms_mean / 1e3) / 1e9
    peak, peak_src = measured_peaks()
    kname = {0: "auto", 1: "flat", 2: "tiles", 3: "flat128", 4: "wide", 5: "bulk"}[kern]
    probe = hbm_copy_probe(dev)

    graph = None
    if args.graph:
        graph = bench_graph(hub, grads, N, E, stream, args.steps)

    # ---- end to end through the public API with host buffers (pinned), H2D/D2H inside
    e2e = None
    if not args.no_e2e:
        e2e = bench_e2e(hub, grads, N, E, Ep, stream, args.e2e_steps, args.e2e_streams)

    cache_table = bench_cache_table(hub, grads, N, E, stream, args) if args.cache_table else None

    cpu = None
    if not args.no_cpu:      # full rounds on all host cores and on one
        cpu = cpu_baseline(mname, N, cb, args.cpu_rounds)

    out = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": round(value / PAPER_GBS, 2), "dtype": "f32", "data": "synthetic",
        "exchanges_per_s": round(N / t_step, 1),
        "config": {"workload": args.config, "keys": len(sizes), "E": E, "E_padded": Ep,
                   "workers": N, "chunk_bytes": cb, "grid": args.grid, "tile_elems": args.tile_elems, "oneshot": args.oneshot,
                   "mode": "M1 (1 GPU, pushes resident, "
                   "zero-copy BORROW)", "kernel": kname, "cache": args.cache,
                   "l2_resident_mib": (None if args.cache != "resident" else
                                       args.resident_mb if args.resident_mb >= 0 else 32),
                   "l2": f"no flush: inputs exceed L2 ({(4 * N + 16) * E / 1e9:.2f} GB/round "
                         f"vs 126 MB L2)" if (4 * N + 16) * E > 4 * 126e6 else
                         "inputs fit in L2 (reported as us/round)",
                   "vs_baseline_basis": "paper PBox ~41.4 GB/s (72.08 exch/s x 574.7 MB, VGG, "
                                        "8 workers; BASELINE.md), other hardware: context"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": ncu_traffic(args.config, kname)[0],
                     "traffic_source": ncu_traffic(args.config, kname)[1],
                     "kernel": "phub_agg_nag (k_flat)", "kernel_ms": round(k_ms_mean, 4),
                     "kernel_ms_min": round(min(k_ms), 4),
                     "kernel_ms_median": round(statistics.median(k_ms), 4),
                     "same_run_hbm_copy_gbs": probe,
                     "frac_of_same_run_copy": round(achieved / probe, 4),
                     "frac_of_8tbs_spec": round(achieved / 8000.0, 4),
                     "algorithmic_bytes_per_launch": algo_bytes,
                     "bytes_per_element": 4 * N + 16, "peak_source": peak_src},
        "clocks": clocks.summary(),
        "gpu_launches": launches,
        "graph": graph,
        "cache_table": cache_table,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(out))
    hub.close()


def bench_graph(hub, grads, N, E, stream, steps, rounds_per_graph=20):
    """Launch-bound configs: the push bookkeeping is host-only, so a round's GPU
    work is one kernel; capture `rounds_per_graph` rounds' kernels in one CUDA
    graph and replay it (the receipts/iteration bookkeeping runs once per
    captured round at capture time, not per replay)."""
    import torch
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(stream)
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(rounds_per_graph):
                for w in range(N):
                    hub.push(w, grads[w])
                hub.aggregate_optimize()
    torch.cuda.synchronize()
    reps = max(1, steps // rounds_per_graph)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / 1e3 / (reps * rounds_per_graph)
    return {"us_per_round": round(t * 1e6, 3), "value": round(N * 4 * E / t / 1e9, 2),
            "unit": "GB/s", "rounds_per_graph": rounds_per_graph, "replays": reps}


def bench_cache_table(hub, grads, N, E, stream, args, reps=20):
    """The caching table of P:913-935 (S 5, "Caching Effectiveness") on B200: the
    fused aggregate + Nesterov kernel under each L2 policy -- cache-enabled (all
    of w' stored evict-last so the pull that follows reads it from L2),
    cache-bypass (every stream evict-first) and resident (a fixed slice of w
    kept in L2 across rounds, the default) -- each timed alone and followed by
    the pull of the whole model (phub_pull ALL_KEYS into a device buffer), plus
    the pull alone ("Opt/Agg Off").  Mean ms over `reps` (CUDA events on the
    launching stream).  The L2 state a policy leaves behind changes the next
    policy's time (profiles/r02_l2/), so each policy is measured after its own
    `settle` rounds; fresh-process numbers are in profiles/r02_l2/."""
    import torch
    from paper_1805_07891_b200 import capi
    dst = torch.empty(hub.E_padded, dtype=torch.float32, device=grads[0].device)
    batch = [(w, capi.PHUB_ALL_KEYS, grads[w]) for w in range(N)]

    def timed(fn):
        for _ in range(3):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    def agg():
        hub.push_batch(batch)
        hub.aggregate_optimize()

    def pull():
        hub.pull(dst)

    def agg_pull():
        agg()
        pull()

    rows = {"pull_only_ms": timed(pull)}
    modes = (("resident", capi.PHUB_CACHE_RESIDENT), ("cached", capi.PHUB_CACHE_ENABLED),
             ("bypass", capi.PHUB_CACHE_BYPASS))
    for mode, val in modes:
        hub.set_option(capi.PHUB_OPT_CACHE, val)
        for _ in range(10):                       # settle: the previous policy's L2 state
            agg()
        rows[f"{mode}_kernel_ms"] = timed(agg)
        rows[f"{mode}_kernel_pull_ms"] = timed(agg_pull)
    hub.set_option(capi.PHUB_OPT_CACHE, capi.PHUB_CACHE_RESIDENT)
    out = {k: round(v, 4) for k, v in rows.items()}
    for mode, _ in modes:
        out[f"{mode}_exchanges_per_s"] = round(N / (rows[f"{mode}_kernel_pull_ms"] / 1e3), 1)
    out["how"] = ("mean of %d rounds each; pull = phub_pull(ALL_KEYS) D2D of the padded model "
                  "(cudaMemcpyAsync: %.0f MB read + written)" % (reps, 4 * hub.E_padded / 1e6))
    return out


def bench_e2e(hub, grads, N, E, Ep, stream, steps, nstreams=1):
    """Same metric through the public C ABI with pinned HOST buffers: every round
    copies the N pushes host->device (PHUB_COPY), runs the kernel, and pulls
    the model back to the host once per worker (PHUB_ALL_KEYS pull, one host
    buffer per worker) -- all inside the timed region.  Rounds are pipelined:
    the H2D pushes of round k+1 (receive slot (k+1) % 2) overlap the D2H pulls
    of round k on the full-duplex PCIe link; each kernel waits for its pushes
    and for the previous round's pulls (it overwrites w).  Copies are spread
    round-robin over `nstreams` streams per direction (several copy engines)."""
    import torch
    host_g = []
    for w in range(N):
        h = torch.empty(Ep, dtype=torch.float32, pin_memory=True)
        h.copy_(grads[w])
        host_g.append(h)
    host_w = [torch.empty(Ep, dtype=torch.float32, pin_memory=True) for _ in range(N)]
    torch.cuda.synchronize()
    K = max(1, int(nstreams))
    s_in = [torch.cuda.Stream() for _ in range(K)]
    s_out = [torch.cuda.Stream() for _ in range(K)]
    s_c = torch.cuda.Stream()
    total = steps + 1

    def ev():
        return torch.cuda.Event(enable_timing=False)

    ev_in = [[ev() for _ in range(K)] for _ in range(total)]
    ev_c = [ev() for _ in range(total)]
    ev_out = [[ev() for _ in range(K)] for _ in range(total)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def round_(k):
        if k >= 2:
            for si in s_in:
                si.wait_event(ev_c[k - 2])         # receive slot k % 2 is free again
        for w in range(N):
            hub.push(w, host_g[w], mode="copy", stream=s_in[w % K])
        for i, si in enumerate(s_in):
            ev_in[k][i].record(si)
            s_c.wait_event(ev_in[k][i])
        if k >= 1:
            for e in ev_out[k - 1]:
                s_c.wait_event(e)                  # previous pulls have read w
        hub.aggregate_optimize(stream=s_c)
        ev_c[k].record(s_c)
        for so in s_out:
            so.wait_event(ev_c[k])
        for w in range(N):
            hub.pull(host_w[w], stream=s_out[w % K])
        for i, so in enumerate(s_out):
            ev_out[k][i].record(so)

    round_(0)                                      # warm-up round
    torch.cuda.synchronize()
    t0.record(s_c)
    for si in s_in + s_out:
        si.wait_event(t0)
    for k in range(1, total):
        round_(k)
    for e in ev_out[total - 1]:
        s_c.wait_event(e)
    t1.record(s_c)
    torch.cuda.synchronize()
    t = t0.elapsed_time(t1) / 1e3 / steps
    probe = pcie_probe(grads[0].device, h_in=host_g[0], h_out=host_w[0])
    probe["fresh_buffers"] = pcie_probe(grads[0].device)
    del host_g, host_w
    per_dir = N * 4 * Ep / t / 1e9
    return {"value": round(N * 4 * E / t / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": N * 4 * Ep, "d2h_bytes_per_step": N * 4 * Ep,
            "steps": steps, "ms_per_step": round(t * 1e3, 3),
            "pcie_probe": probe, "gbs_per_direction": round(per_dir, 2),
            "frac_of_pcie_bidir": round(per_dir / probe["bidir_gbs_per_direction"], 4),
            "path": f"phub_push(PHUB_COPY, pinned host) x N -> phub_aggregate_optimize -> "
                    f"phub_pull(host) x N; rounds pipelined (H2D of k+1 || D2H of k), copies "
                    f"on {K} stream(s) per direction"}


if __name__ == "__main__":
    main()
