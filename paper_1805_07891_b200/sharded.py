"""Chunks sharded by owner over the GPUs of one box (PAPER.md P:708-717,
P:743 "micro-shards inside a box").

One process per GPU.  Rank r owns the CONTIG chunk range [b_r, e_r) of the
padded layout (chunk granular, reading R10) and hosts workers
[r*N/G, (r+1)*N/G) -- contiguous blocks, so rank order is worker order.

A round (mode M3) is:
  push   every hosted worker's slice [b_o, e_o) goes to owner o: one NCCL group
         of send/recv (a reduce-scatter by transport, not ncclReduceScatter, so
         the owner still sums in worker-id order, reading R3);
  agg    the owner's fused sm_100a kernel over its range (libphub);
  pull   the owners' updated ranges are exchanged in one NCCL group
         (all-gather-v) straight into every rank's weight replica.

torch.distributed is plumbing only (device memory, streams, the NCCL group);
the exchange schedule below is device-agnostic so the host logic runs under
gloo on CPU in the tests.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import capi


@dataclass
class ExchangePlan:
    """Who sends which padded slice to whom (pure host logic)."""
    rank: int
    world: int
    num_workers: int
    E_padded: int
    ranges: list            # [(begin, end)] per owner, abutting, covering [0, E_padded)

    @classmethod
    def build(cls, key_sizes, num_workers, chunk_size_bytes, rank, world):
        if num_workers % world != 0:
            raise ValueError(f"{num_workers} workers cannot be hosted evenly on {world} ranks")
        Ep, _offs, ranges = capi.phub_plan_ranges(key_sizes, chunk_size_bytes, world)
        return cls(rank, world, num_workers, Ep, ranges)

    @property
    def per_rank(self):
        return self.num_workers // self.world

    def host_of(self, worker):
        return worker // self.per_rank

    def hosted(self, rank=None):
        r = self.rank if rank is None else rank
        return list(range(r * self.per_rank, (r + 1) * self.per_rank))

    def owned(self, rank=None):
        return self.ranges[self.rank if rank is None else rank]

    def nvlink_bytes_out(self):
        """Bytes this rank sends per round (push slices + pulled range copies)."""
        b, e = self.owned()
        push = sum(4 * (oe - ob) for o, (ob, oe) in enumerate(self.ranges) if o != self.rank) \
            * self.per_rank
        pull = 4 * (e - b) * (self.world - 1)
        return push + pull

    def nvlink_bytes_in(self):
        b, e = self.owned()
        push = 4 * (e - b) * (self.num_workers - self.per_rank)
        pull = sum(4 * (oe - ob) for o, (ob, oe) in enumerate(self.ranges) if o != self.rank)
        return push + pull


def push_exchange(plan: ExchangePlan, grads: dict, recv: dict, group=None):
    """Send hosted workers' owner slices; receive remote workers' slices of the
    owned range into recv[w] (length e_r - b_r).  Returns after the receives
    are ordered before later work on the current stream."""
    import torch.distributed as dist
    ops = []
    for w in plan.hosted():
        for o, (b, e) in enumerate(plan.ranges):
            if o != plan.rank and e > b:
                ops.append(dist.P2POp(dist.isend, grads[w][b:e], o, group))
    b, e = plan.owned()
    if e > b:
        for w in range(plan.num_workers):
            if plan.host_of(w) != plan.rank:
                ops.append(dist.P2POp(dist.irecv, recv[w], plan.host_of(w), group))
    if ops:
        for work in dist.batch_isend_irecv(ops):
            work.wait()


def pull_exchange(plan: ExchangePlan, replica, group=None):
    """All-gather-v of the owners' updated ranges into every rank's replica."""
    import torch.distributed as dist
    ops = []
    b, e = plan.owned()
    for p in range(plan.world):
        if p == plan.rank:
            continue
        if e > b:
            ops.append(dist.P2POp(dist.isend, replica[b:e], p, group))
        pb, pe = plan.ranges[p]
        if pe > pb:
            ops.append(dist.P2POp(dist.irecv, replica[pb:pe], p, group))
    if ops:
        for work in dist.batch_isend_irecv(ops):
            work.wait()


class ShardedPHub:
    """The sharded parameter exchange on this rank's GPU (public multi-GPU API).

        sh = ShardedPHub(key_sizes, num_workers=8)        # after init_process_group("nccl")
        sh.exchange({w: grad_w for w in sh.hosted})        # push -> aggregate -> pull
        sh.weights()                                       # full updated replica (padded)
    """

    def __init__(self, key_sizes, num_workers, chunk_size_bytes=32768, lr=0.1, momentum=0.9,
                 rescale=0.0, device=None, group=None):
        import torch
        import torch.distributed as dist
        from .phub import PHub
        self.group = group
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.plan = ExchangePlan.build(key_sizes, num_workers, chunk_size_bytes, rank, world)
        self.hub = PHub(key_sizes, num_workers, chunk_size_bytes=chunk_size_bytes, lr=lr,
                        momentum=momentum, rescale=rescale, device=self.device,
                        num_owners=world, owner_rank=rank, owner_policy="contig")
        assert self.hub.E_padded == self.plan.E_padded
        assert tuple(self.hub.owner_range()) == tuple(self.plan.owned())
        b, e = self.plan.owned()
        self.recv = {w: torch.empty(e - b, dtype=torch.float32, device=self.device)
                     for w in range(num_workers) if self.plan.host_of(w) != rank}
        self.replica = self.hub.weights()

    @property
    def hosted(self):
        return self.plan.hosted()

    def push(self, grads: dict):
        push_exchange(self.plan, grads, self.recv, self.group)
        for w in range(self.plan.num_workers):
            if self.plan.host_of(w) == self.plan.rank:
                self.hub.push(w, grads[w], key=capi.PHUB_ALL_KEYS)       # own slice, zero copy
            else:
                self.hub.push(w, self.recv[w], key=capi.PHUB_OWNED_RANGE)

    def aggregate_optimize(self):
        self.hub.aggregate_optimize()

    def pull(self):
        pull_exchange(self.plan, self.replica, self.group)

    def exchange(self, grads: dict):
        self.push(grads)
        self.aggregate_optimize()
        self.pull()

    def exchange_host(self, host_grads: dict, dev_grads: dict, host_out: dict):
        """End-to-end round from host memory: H2D copy of each hosted worker's
        gradient (pinned host -> device staging), the exchange, and a D2H copy
        of the updated replica for each hosted worker."""
        for w in self.hosted:
            dev_grads[w].copy_(host_grads[w], non_blocking=True)
        self.exchange(dev_grads)
        for w in self.hosted:
            host_out[w].copy_(self.replica, non_blocking=True)

    def weights(self):
        return self.replica

    def close(self):
        self.hub.close()


class PeerMappingError(RuntimeError):
    """CUDA IPC peer mapping is unavailable on at least one rank (all ranks raise)."""


class P2PShardedPHub:
    """Peer-memory form of the sharded exchange: ONE kernel
    per round on each owner reads its workers' slices straight out of the
    peers' gradient buffers over NVLink (in worker-id order, so the sum stays
    bit-exact), applies Nesterov, and stores w' into its own replica and into
    every peer replica -- push, aggregate+optimize and the pull's all-gather
    fused, no NCCL data movement.

    Hosted workers write their gradients into ``gradients()[w]`` (buffers
    allocated by libphub so they can be exported with CUDA IPC).  Rounds are
    ordered across GPUs by a stream-ordered NCCL barrier (a 1-element
    all-reduce) before and after the kernel; no kernel ever spins on a peer.
    """

    def __init__(self, key_sizes, num_workers, chunk_size_bytes=32768, lr=0.1, momentum=0.9,
                 rescale=0.0, device=None, group=None, nslots=2):
        import torch
        import torch.distributed as dist
        from .phub import PHub, _CudaArray
        self.group = group
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.plan = ExchangePlan.build(key_sizes, num_workers, chunk_size_bytes, rank, world)
        self.hub = PHub(key_sizes, num_workers, chunk_size_bytes=chunk_size_bytes, lr=lr,
                        momentum=momentum, rescale=rescale, device=self.device,
                        num_owners=world, owner_rank=rank, owner_policy="contig")
        Ep = self.hub.E_padded
        dev = self.device
        # gradient buffers per (slot, worker): two slots let round k+1's gradients
        # be written while round k's exchange still reads slot k % 2
        self.nslots = int(nslots)
        self._own = {(sl, w): capi.phub_alloc_shared(dev, 4 * Ep)
                     for sl in range(self.nslots) for w in self.plan.hosted()}
        self._grads = {key: torch.as_tensor(_CudaArray(p, Ep, self), device=f"cuda:{dev}")
                       for key, p in self._own.items()}
        for t in self._grads.values():
            t.zero_()
        mine = (rank, {key: capi.phub_ipc_get_handle(dev, p) for key, p in self._own.items()},
                capi.phub_ipc_get_handle(dev, self.hub.weights_ptr()))
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        self._peer_grad, self._peer_w = {}, []
        err = None
        try:
            for r, hs, wh in sorted(allh, key=lambda x: x[0]):
                if r == rank:
                    continue
                for key, h in hs.items():
                    self._peer_grad[key] = capi.phub_ipc_open(dev, h)
                self._peer_w.append(capi.phub_ipc_open(dev, wh))
            capi.phub_set_replicas(self.hub.ctx, self._peer_w)
        except capi.PhubError as e:
            err = e
        # every rank must agree before anyone relies on peer mappings
        ok = torch.tensor([0 if err else 1], dtype=torch.int32, device=f"cuda:{dev}")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            for p in list(self._peer_grad.values()) + self._peer_w:
                try:
                    capi.phub_ipc_close(dev, p)
                except capi.PhubError:
                    pass
            self._grads = {}
            for p in self._own.values():
                capi.phub_free_shared(dev, p)
            self.hub.close()
            raise PeerMappingError(f"peer mapping failed on some rank ({err or 'other rank'})")
        self._flag = torch.zeros(1, dtype=torch.float32, device=f"cuda:{dev}")
        self.replica = self.hub.weights()
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)

    @property
    def hosted(self):
        return self.plan.hosted()

    def gradients(self, slot: int = 0) -> dict:
        """Device buffers (padded layout) the hosted workers write their gradients into."""
        return {w: self._grads[(slot, w)] for w in self.hosted}

    def barrier(self):
        import torch.distributed as dist
        dist.all_reduce(self._flag, group=self.group)

    def push(self, slot: int = 0):
        Ep = self.hub.E_padded
        for w in range(self.plan.num_workers):
            key = (slot, w)
            ptr = self._own[key] if key in self._own else self._peer_grad[key]
            self.hub.push(w, ptr, key=capi.PHUB_ALL_KEYS, mode="borrow", n=Ep)

    def exchange(self, slot: int = 0):
        self.barrier()                  # every rank's gradients of this round are in place
        self.push(slot)                 # zero-copy: local and peer-mapped pointers
        self.hub.aggregate_optimize()   # NVLink loads + NAG + NVLink replica stores
        self.barrier()                  # every owner's stores into this replica are done

    def exchange_host(self, host_grads: dict, host_out: dict, slot: int = 0):
        g = self.gradients(slot)
        for w in self.hosted:
            g[w].copy_(host_grads[w], non_blocking=True)
        self.exchange(slot)
        for w in self.hosted:
            host_out[w].copy_(self.replica, non_blocking=True)

    def weights(self):
        return self.replica

    def close(self):
        import torch
        import torch.distributed as dist
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        capi.phub_set_replicas(self.hub.ctx, [])
        for p in list(self._peer_grad.values()) + self._peer_w:
            capi.phub_ipc_close(self.device, p)
        dist.barrier(group=self.group)
        self._grads = {}
        for p in self._own.values():
            capi.phub_free_shared(self.device, p)
        self._own = {}
        self.hub.close()


class AllReduceBaseline:
    """Comparison baseline (the paper's Gloo comparison,
    P:1080-1085: "we ran our SGD/Nesterov optimizer on all nodes after
    reduction"): every GPU sums its hosted workers, NCCL all-reduces the sums
    (ring/tree/NVLS order -- NOT worker order, so results match the oracle only
    within rounding, reading R3), then runs the Nesterov step on the WHOLE model
    (libphub kernel with one pushed gradient, rescale 1/N).  Not the product
    path; it exists to be measured against it."""

    def __init__(self, key_sizes, num_workers, chunk_size_bytes=32768, lr=0.1, momentum=0.9,
                 device=None, group=None):
        import torch
        import torch.distributed as dist
        from .phub import PHub
        self.group = group
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.plan = ExchangePlan.build(key_sizes, num_workers, chunk_size_bytes, rank, world)
        self.hub = PHub(key_sizes, 1, chunk_size_bytes=chunk_size_bytes, lr=lr,
                        momentum=momentum, rescale=1.0 / num_workers, device=self.device)
        self.sum = torch.zeros(self.hub.E_padded, dtype=torch.float32,
                               device=f"cuda:{self.device}")
        self.replica = self.hub.weights()

    @property
    def hosted(self):
        return self.plan.hosted()

    def exchange(self, grads: dict):
        import torch.distributed as dist
        hosted = self.hosted
        self.sum.copy_(grads[hosted[0]])
        for w in hosted[1:]:
            self.sum.add_(grads[w])
        dist.all_reduce(self.sum, group=self.group)
        self.hub.push(0, self.sum)
        self.hub.aggregate_optimize()

    def weights(self):
        return self.replica

    def close(self):
        self.hub.close()


def chain_pieces(E_padded: int, pieces: int):
    """Pipeline pieces of the chained exchange: <= `pieces` abutting ranges
    covering [0, E_padded), boundaries on 64-element (256 B) multiples."""
    k = max(1, int(pieces))
    step = -(-E_padded // k)
    step = -(-step // 64) * 64
    return [(b, min(E_padded, b + step)) for b in range(0, E_padded, step)]


def chain_nvlink_bytes(E_padded: int, world: int, rank: int):
    """(out, in) NVLink bytes of one chained round for `rank`: one partial per
    link, and the last rank's w' stores into the other replicas."""
    out = 4 * E_padded * ((world - 1) if rank == world - 1 else 1)
    inn = 4 * E_padded * ((1 if rank > 0 else 0) + (1 if rank < world - 1 else 0))
    return out, inn


def chain_block_for(E_padded: int) -> int:
    """Block size of the block-streamed chain (elements): 8K blocks up to 64 M
    elements, 12K above -- measured optimum at G = 2 (profiles/r01_chain_blocks:
    ResNet-50 / AlexNet best at 8K, VGG-19 at 12K; smaller blocks pay the
    per-block fence, larger ones the pipeline fill)."""
    return 8192 if E_padded < (64 << 20) else 12288


class ExchangeFailed(RuntimeError):
    """A device-side flag wait of this job expired on this rank (PHUB_ERR_SYNC_TIMEOUT):
    the round is incomplete.  Raised by exchange() on every later round; the rank
    still takes part in the round's collectives first, so its peers never hang --
    their waits on its flags expire and their next exchange() raises too."""


class _DeviceWaitExchange:
    """Shared failure handling of the exchanges whose kernels wait on device flags
    (chain, push, hierarchical): a failed context skips its kernels but keeps
    every collective of the round, then raises."""

    def barrier(self):
        """Stream-ordered one-float all-reduce (counted, see _round)."""
        import torch.distributed as dist
        self._nbar = getattr(self, "_nbar", 0) + 1
        dist.all_reduce(self._flag, group=self.group)

    def _barriers_per_round(self):
        return 2                                   # start + end

    def _round(self, body):
        """Run one round's body; if the context is (or becomes) failed, still issue
        the round's remaining collectives, then raise ExchangeFailed."""
        self._nbar = 0
        st = capi.phub_check(self.hub.ctx)
        if not st:
            try:
                body()
                return
            except capi.PhubError as e:
                st = e.status
        for _ in range(self._barriers_per_round() - self._nbar):
            self.barrier()
        raise ExchangeFailed(f"rank {self.rank}: {capi.STATUS_NAMES[st]} "
                             f"({capi.phub_last_error(self.hub.ctx)})")

    def check(self):
        """Collective: wait for this rank's work and raise ExchangeFailed on EVERY
        rank if any rank's context failed (its round results are incomplete)."""
        import torch
        import torch.distributed as dist
        try:
            self.hub.synchronize()
            st = 0
        except capi.PhubError as e:
            st = e.status
        t = torch.tensor([st], dtype=torch.int32, device=f"cuda:{self.device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        worst = int(t.item())
        if worst:
            raise ExchangeFailed(f"an exchange failed on some rank: {capi.STATUS_NAMES[worst]}")

    def sync_timeouts(self) -> int:
        return capi.phub_sync_timeouts(self.hub.ctx)


class ChainShardedPHub(_DeviceWaitExchange):
    """Chained exchange.

    Workers are hosted in rank order, so the worker-order sum can be built
    rank by rank: rank p adds its hosted workers to the partial sum of ranks
    0..p-1 (phub_partial_sum); the last rank finishes the sum, runs the fused
    Nesterov kernel on the whole model (phub_aggregate_range) and stores w'
    into every replica.  Because every partial starts from +0 and adds in
    order, the result is bit-identical to the one-GPU sum (R3, R4).

    Each link carries one model-size partial per round (4E bytes) instead of
    N/G gradient slices per owner -- fewer NVLink bytes than the sharded
    exchange when G is small (G = 2: 4E per direction vs 10E).

    sync="blocks" (default): ONE persistent launch per rank and round; the
      model is cut into blocks of `block` elements with one device flag each,
      so rank p+1 starts on block b as soon as rank p has stored it into its
      inbox over NVLink and raised the flag (streaming).
    sync="flags": the model is split into `pieces`, one launch per piece, each
      waiting for a per-piece flag (device-side) -- the previous design.
    sync="barrier": per-piece launches separated by NCCL barriers.
    """

    def __init__(self, key_sizes, num_workers, chunk_size_bytes=32768, lr=0.1, momentum=0.9,
                 device=None, group=None, pieces=8, sync="blocks", nslots=2, block=0):
        import torch
        import torch.distributed as dist
        from .phub import PHub, _CudaArray
        self.group = group
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        self.rank, self.world = rank, world
        if sync not in ("blocks", "flags", "barrier"):
            raise ValueError("sync must be 'blocks', 'flags' or 'barrier'")
        self.sync = sync
        self.block = int(block)          # 0: chosen from the model size below
        self._epoch = 0
        self.device = torch.cuda.current_device() if device is None else int(device)
        dev = self.device
        self.plan = ExchangePlan.build(key_sizes, num_workers, chunk_size_bytes, rank, world)
        self.last = rank == world - 1
        per = num_workers // world
        if self.last:      # the finishing rank: incoming partial + its own workers
            nw = per + (1 if world > 1 else 0)
            self.hub = PHub(key_sizes, nw, chunk_size_bytes=chunk_size_bytes, lr=lr,
                            momentum=momentum, rescale=1.0 / num_workers, device=dev)
        else:              # a summing rank: its context is used for partial sums + its replica
            self.hub = PHub(key_sizes, per, chunk_size_bytes=chunk_size_bytes, lr=lr,
                            momentum=momentum, device=dev)
        Ep = self.hub.E_padded
        if self.block <= 0:
            self.block = chain_block_for(Ep)
        self.nslots = int(nslots)
        self._own = {(sl, w): capi.phub_alloc_shared(dev, 4 * Ep)
                     for sl in range(self.nslots) for w in self.plan.hosted()}
        self._grads = {key: torch.as_tensor(_CudaArray(p, Ep, self), device=f"cuda:{dev}")
                       for key, p in self._own.items()}
        for t in self._grads.values():
            t.zero_()
        # the incoming partial sum: an inbox on every rank > 0, stored into by rank - 1
        self._pin = capi.phub_alloc_shared(dev, 4 * Ep) if rank > 0 else None
        self.pieces = chain_pieces(Ep, pieces)
        nflags = -(-Ep // self.block) if sync == "blocks" else len(self.pieces)
        # one uint32 "ready" flag per block (or piece), raised by the previous rank
        self._flags = capi.phub_alloc_shared(dev, 4 * nflags) if rank > 0 else None
        if self._flags:
            torch.as_tensor(_CudaArray(self._flags, nflags, self), device=f"cuda:{dev}").zero_()
        h = capi.phub_ipc_get_handle
        mine = (rank, h(dev, self._pin) if self._pin else None,
                h(dev, self.hub.weights_ptr()),
                h(dev, self._flags) if self._flags else None)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        allh.sort(key=lambda x: x[0])
        self._opened = []
        self._next_in = self._next_flags = None

        def open_(hd):
            p_ = capi.phub_ipc_open(dev, hd)
            self._opened.append(p_)
            return p_

        err = None
        try:
            if not self.last:
                self._next_in = open_(allh[rank + 1][1])
                self._next_flags = open_(allh[rank + 1][3])
            if self.last:
                reps = [open_(wh) for r, _pin, wh, _fl in allh if r != rank]
                capi.phub_set_replicas(self.hub.ctx, reps)
        except capi.PhubError as ex:
            err = ex
        # every rank must agree before anyone relies on peer mappings
        ok = torch.tensor([0 if err else 1], dtype=torch.int32, device=f"cuda:{dev}")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            for p_ in self._opened:
                try:
                    capi.phub_ipc_close(dev, p_)
                except capi.PhubError:
                    pass
            self._grads = {}
            for p_ in list(self._own.values()) + [x for x in (self._pin, self._flags) if x]:
                capi.phub_free_shared(dev, p_)
            self.hub.close()
            raise PeerMappingError(f"peer mapping failed on some rank ({err or 'other rank'})")
        self._flag = torch.zeros(1, dtype=torch.float32, device=f"cuda:{dev}")
        self.replica = self.hub.weights()
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)

    @property
    def hosted(self):
        return self.plan.hosted()

    def gradients(self, slot: int = 0) -> dict:
        return {w: self._grads[(slot, w)] for w in self.hosted}

    def _barriers_per_round(self):
        return 2 if self.sync != "barrier" else len(self.pieces) + self.world - 1

    def exchange(self, slot: int = 0):
        """One round: push -> aggregate + Nesterov -> replicas.  Raises
        ExchangeFailed if this rank's context failed."""
        self._round(lambda: self._exchange(slot))

    def _exchange(self, slot):
        Ep = self.hub.E_padded
        hosted = self.hosted
        upstream = self._pin                                       # partial of ranks 0..p-1
        if self.sync != "barrier":
            # start barrier: the last rank's kernel stores w' into every other rank's
            # replica, so every rank must be done reading its replica (e.g. the
            # previous round's pull, enqueued after that round's end barrier) first
            self.barrier()
        if self.last:
            w0 = 0
            if self.world > 1:
                self.hub.push(0, upstream, mode="borrow", n=Ep)
                w0 = 1
            for i, w in enumerate(hosted):
                self.hub.push(w0 + i, self._own[(slot, w)], mode="borrow", n=Ep)
        srcs = ([upstream] if upstream else []) + [self._own[(slot, w)] for w in hosted]
        stream = self.hub._stream(None)
        K = len(self.pieces)
        if self.sync == "blocks":
            # one persistent launch per rank: per-block flags order the stages
            self._epoch += 1
            ep = self._epoch
            wait = (self._flags, ep) if self._flags else None
            if self.last:
                capi.phub_aggregate_range(self.hub.ctx, 0, Ep, stream, wait=wait, block=self.block)
            else:
                capi.phub_partial_sum(self.hub.ctx, srcs, self._next_in, 0, Ep, stream, wait=wait,
                                      signal=(self._next_flags, ep), block=self.block)
            self.barrier()                   # replicas complete; buffers free for the next round
            return
        if self.sync == "flags":
            # all pieces enqueued at once; each launch waits (on the device) for the
            # previous rank's "piece ready" flag and raises the next rank's
            self._epoch += 1
            ep = self._epoch
            for p, (b, e) in enumerate(self.pieces):
                wait = (self._flags + 4 * p, ep) if self._flags else None
                if self.last:
                    capi.phub_aggregate_range(self.hub.ctx, b, e, stream, wait=wait)
                else:
                    capi.phub_partial_sum(self.hub.ctx, srcs, self._next_in, b, e, stream,
                                          wait=wait, signal=(self._next_flags + 4 * p, ep))
            self.barrier()                   # replicas complete; buffers free for the next round
            return
        for j in range(K + self.world - 1):
            p = j - self.rank
            if 0 <= p < K:
                b, e = self.pieces[p]
                if self.last:
                    capi.phub_aggregate_range(self.hub.ctx, b, e, stream)
                else:
                    capi.phub_partial_sum(self.hub.ctx, srcs, self._next_in, b, e, stream)
            self.barrier()                   # piece p is complete before the next rank reads it

    def exchange_host(self, host_grads: dict, host_out: dict, slot: int = 0):
        g = self.gradients(slot)
        for w in self.hosted:
            g[w].copy_(host_grads[w], non_blocking=True)
        self.exchange(slot)
        for w in self.hosted:
            host_out[w].copy_(self.replica, non_blocking=True)

    def weights(self):
        return self.replica

    def close(self):
        import torch
        import torch.distributed as dist
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        if self.last:
            capi.phub_set_replicas(self.hub.ctx, [])
        for p in self._opened:
            capi.phub_ipc_close(self.device, p)
        dist.barrier(group=self.group)
        self._grads = {}
        for p in self._own.values():
            capi.phub_free_shared(self.device, p)
        if self._pin:
            capi.phub_free_shared(self.device, self._pin)
        if self._flags:
            capi.phub_free_shared(self.device, self._flags)
        self._own = {}
        self.hub.close()


def hier_slot(slot: int, src_rack: int, racks: int, owned: int) -> int:
    """Element offset, inside an owner's inbox allocation (2 x racks x owned
    elements), of the slot that rack `src_rack` fills in epoch parity `slot`.
    Producer and consumer both address the inbox through this function."""
    return (slot * racks + src_rack) * owned


def hier_nvlink_bytes(ranges, E_padded: int, rank: int):
    """(out, in) NVLink bytes of one hierarchical round for `rank`: its rack
    aggregate of every other owner's range out and the w' of its own range to
    the other racks' replicas; symmetric inbound."""
    b, e = ranges[rank]
    G = len(ranges)
    out = 4 * (E_padded - (e - b)) + 4 * (e - b) * (G - 1)
    inn = 4 * (e - b) * (G - 1) + 4 * (E_padded - (e - b))
    return out, inn


class HierPHub(_DeviceWaitExchange):
    """Hierarchical reduction across racks (PAPER.md
    P:746-763, emulated in P:1002-1012).

    Every GPU is one rack's PBox with its own `workers_per_rack` workers (their
    gradients resident in its HBM, like the 1-GPU job).  One round is the
    paper's three steps, fused in ONE persistent launch per GPU
    (phub_hier_exchange): the rack aggregate of the local workers, the
    cross-rack aggregation in rack order over NVLink (each GPU stores its rack
    aggregate of every other owner's range straight into that owner's inbox),
    and the Nesterov step on the owned range with w' stored into every rack's
    weight replica (the per-rack broadcast).  Per-GPU work is fixed as racks are
    added (weak scaling); the cross-rack traffic per GPU is 2(G-1)/G model
    sizes, independent of the number of workers per rack -- the "1/N
    cross-rack traffic" the paper trades rounds for.
    """

    def __init__(self, key_sizes, workers_per_rack=8, chunk_size_bytes=32768, lr=0.1,
                 momentum=0.9, device=None, group=None, block=32768, nslots=2,
                 worker_order=False, device_barrier=True):
        import torch
        import torch.distributed as dist
        from .phub import PHub, _CudaArray
        self.group = group
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        self.R, self.rack, self.P = world, rank, int(workers_per_rack)
        self.rank = rank
        self.block = int(block)
        # worker_order: the flat worker-order sum of one job's R x P workers (raw
        # slices pushed to the owners) instead of the rack-grouped sum
        self.worker_order = bool(worker_order)
        # round barriers inside the launch (phub_hier.device_barrier) instead of two
        # NCCL all-reduces per round
        self.device_barrier = bool(device_barrier) and world > 1
        S = self.P if self.worker_order else 1          # slices per (slot, source rack)
        self.device = torch.cuda.current_device() if device is None else int(device)
        dev = self.device
        self.hub = PHub(key_sizes, self.P, chunk_size_bytes=chunk_size_bytes, lr=lr,
                        momentum=momentum, rescale=1.0 / (self.R * self.P), device=dev,
                        num_owners=world, owner_rank=rank, owner_policy="contig")
        Ep = self.hub.E_padded
        b, e = self.hub.owner_range()
        L = e - b
        self.nslots = int(nslots)
        self._own = {(sl, k): capi.phub_alloc_shared(dev, 4 * Ep)
                     for sl in range(self.nslots) for k in range(self.P)}
        self._grads = {key: torch.as_tensor(_CudaArray(p, Ep, self), device=f"cuda:{dev}")
                       for key, p in self._own.items()}
        for t in self._grads.values():
            t.zero_()
        # inbox: 2 epoch-parity slots x R source racks x S slices x L owned elements
        self._inbox = capi.phub_alloc_shared(dev, 4 * 2 * world * S * max(L, 1))
        # block flags sized by the LARGEST owner range (J blocks) on every rack, then
        # the 2 x world round-barrier flags (phub_hier.device_barrier)
        J = max(max(1, -(-(oe - ob) // self.block)) for ob, oe in
                (self.hub.owner_range(o) for o in range(world)))
        nfl = J * world + 2 * world
        self._flags = capi.phub_alloc_shared(dev, 4 * nfl)
        torch.as_tensor(_CudaArray(self._flags, nfl, self), device=f"cuda:{dev}").zero_()
        h = capi.phub_ipc_get_handle
        mine = (rank, b, e, h(dev, self._inbox), h(dev, self._flags),
                h(dev, self.hub.weights_ptr()))
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        allh.sort(key=lambda x: x[0])
        self._opened = []
        self.inbox = [[0] * world for _ in range(2)]
        self.peer_inbox = [[0] * world for _ in range(2)]
        self.peer_flags = [0] * world
        reps = []
        err = None
        try:
            for o, ob, oe, ih, fh, wh in allh:
                if o == rank:
                    continue
                for hd in (ih, fh, wh):
                    self._opened.append(capi.phub_ipc_open(dev, hd))
                pin, pfl, pw = self._opened[-3:]
                reps.append(pw)
                self.peer_flags[o] = pfl
                for sl in range(2):
                    # padded-based: ptr + 4x addresses element x of o's range in o's slot for us
                    self.peer_inbox[sl][o] = pin + 4 * hier_slot(sl, rank, world, S * (oe - ob)) \
                        - 4 * ob
                    self.inbox[sl][o] = self._inbox + 4 * hier_slot(sl, o, world, S * L) - 4 * b
            capi.phub_set_replicas(self.hub.ctx, reps)
        except capi.PhubError as ex:
            err = ex
        # every rank must agree before anyone relies on peer mappings
        ok = torch.tensor([0 if err else 1], dtype=torch.int32, device=f"cuda:{dev}")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            for p_ in self._opened:
                try:
                    capi.phub_ipc_close(dev, p_)
                except capi.PhubError:
                    pass
            self._grads = {}
            for p_ in list(self._own.values()) + [self._inbox, self._flags]:
                capi.phub_free_shared(dev, p_)
            self.hub.close()
            raise PeerMappingError(f"peer mapping failed on some rank ({err or 'other rank'})")
        self.epoch = 0
        self._flag = torch.zeros(1, dtype=torch.float32, device=f"cuda:{dev}")
        self.replica = self.hub.weights()      # this rank's full replica (padded layout)
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)

    @property
    def num_workers(self):
        return self.R * self.P

    @property
    def hosted(self):
        """Local worker indices of this rack (0..P-1)."""
        return list(range(self.P))

    def exchange_host(self, host_grads: dict, host_out: dict, slot: int = 0):
        g = self.gradients(slot)
        for k in self.hosted:
            g[k].copy_(host_grads[k], non_blocking=True)
        self.exchange(slot)
        for k in self.hosted:
            host_out[k].copy_(self.replica, non_blocking=True)

    def gradients(self, slot: int = 0) -> dict:
        """This rack's gradient buffers (padded layout), keyed by local worker index."""
        return {k: self._grads[(slot, k)] for k in range(self.P)}

    def exchange(self, slot: int = 0):
        """One round in one launch per GPU.  Raises ExchangeFailed if this rank's
        context failed."""
        self._round(lambda: self._exchange(slot))

    def _barriers_per_round(self):
        return 0 if self.device_barrier else 2

    def _exchange(self, slot):
        Ep = self.hub.E_padded
        # start barrier: this round's kernels store w' into every rank's replica,
        # so every rank must be done reading its replica from the previous round
        # (e.g. a pull enqueued after that round's end barrier) -- in-kernel flags
        # with device_barrier (the launch is stream-ordered after those reads)
        if not self.device_barrier:
            self.barrier()
        for k in range(self.P):
            self.hub.push(k, self._own[(slot, k)], mode="borrow", n=Ep)
        self.epoch += 1
        par = self.epoch % 2
        capi.phub_hier_exchange(self.hub.ctx, self.R, self.block, self.inbox[par],
                                self.peer_inbox[par], self._flags, self.peer_flags, self.epoch,
                                self.hub._stream(None), worker_order=self.worker_order,
                                device_barrier=self.device_barrier)
        if not self.device_barrier:
            self.barrier()                   # every rack's w' stores into this replica are done

    def weights(self):
        return self.replica

    def close(self):
        import torch
        import torch.distributed as dist
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        capi.phub_set_replicas(self.hub.ctx, [])
        for p in self._opened:
            capi.phub_ipc_close(self.device, p)
        dist.barrier(group=self.group)
        self._grads = {}
        for p in self._own.values():
            capi.phub_free_shared(self.device, p)
        capi.phub_free_shared(self.device, self._inbox)
        capi.phub_free_shared(self.device, self._flags)
        self._own = {}
        self.hub.close()


class PushShardedPHub(HierPHub):
    """Owner-sharded exchange of the N-worker job with every NVLink transfer a
    store (all-to-all SM stores run at ~680 GB/s per direction,
    loads mixed with stores on the same links at ~600-670): one launch per GPU
    (phub_hier_exchange, worker_order) stores each hosted worker's raw slice
    of every other owner's range into that owner's inbox, and sums its own
    range over all N workers in worker order (R3; bit-identical to the 1-GPU
    sum) -> Nesterov -> w' into every replica.  Workers are hosted in rank
    order: rank r hosts global workers [r*N/G, (r+1)*N/G).  Same interface as
    P2PShardedPHub (gradients() keyed by global worker id)."""

    def __init__(self, key_sizes, num_workers, chunk_size_bytes=32768, lr=0.1, momentum=0.9,
                 device=None, group=None, block=12288, nslots=2, device_barrier=True):
        import torch.distributed as dist
        world = dist.get_world_size(group)
        if num_workers % world:
            raise ValueError(f"{num_workers} workers cannot be hosted evenly on {world} ranks")
        super().__init__(key_sizes, workers_per_rack=num_workers // world,
                         chunk_size_bytes=chunk_size_bytes, lr=lr, momentum=momentum,
                         device=device, group=group, block=block, nslots=nslots,
                         worker_order=True, device_barrier=device_barrier)
        self.plan = ExchangePlan.build(key_sizes, num_workers, chunk_size_bytes, self.rack, world)

    @property
    def hosted(self):
        return [self.rack * self.P + k for k in range(self.P)]

    def gradients(self, slot: int = 0) -> dict:
        return {self.rack * self.P + k: self._grads[(slot, k)] for k in range(self.P)}

    def exchange_host(self, host_grads: dict, host_out: dict, slot: int = 0):
        g = self.gradients(slot)
        for w in self.hosted:
            g[w].copy_(host_grads[w], non_blocking=True)
        self.exchange(slot)
        for w in self.hosted:
            host_out[w].copy_(self.replica, non_blocking=True)


# ------------------------------------------------- scheduled exchange (8.6)
# Owner weights and RAW fractions per G (W = 8/G workers per GPU) from the
# byte-balancing model of scripts/sched_lp.py: the busiest NVLink port moves
# 1.000 / 1.769 / 1.789 / 1.750 model sizes at G = 2 / 3 / 4 / 8, vs 2.500 /
# 2.667 / 2.250 / 1.750 for the push exchange (all RAW).
SCHED_TABLE = {
    2: ([0.0, 1.0], [0.0, 0.0]),
    3: ([0.3846, 0.1538, 0.4616], [0.4, 0.0, 0.1667]),
    4: ([0.2982, 0.193, 0.193, 0.3158], [0.5294, 0.0, 0.0, 0.1667]),
    8: ([0.125] * 8, [1.0] * 8),
}


def sched_port_bytes(G: int, W: int, weights, raw_frac):
    """Busiest-direction bytes (in model sizes) of every GPU's NVLink port for
    owner shares `weights` and RAW fractions `raw_frac` (scripts/sched_lp.py's
    byte model, plain Python): RAW -- W raw slices from every other rank into
    the owner; CHAIN -- one partial per hop 0 -> 1 -> ... -> G-1, plus the
    finished sum into the owner unless it is the last rank; w' of every share
    into every other replica."""
    inn, out = [0.0] * G, [0.0] * G
    for o in range(G):
        raw, ch = weights[o] * raw_frac[o], weights[o] * (1.0 - raw_frac[o])
        for q in range(G):
            if q != o:
                inn[o] += W * raw
                out[q] += W * raw
                out[o] += weights[o]          # replica stores
                inn[q] += weights[o]
        for p in range(G - 1):
            out[p] += ch
            inn[p + 1] += ch
        if o != G - 1:
            out[G - 1] += ch
            inn[o] += ch
    return [max(i, x) for i, x in zip(inn, out)]


def sched_nvlink_bytes(bounds, split, W: int, rank: int):
    """(out, in) NVLink bytes of `rank` per round of the scheduled exchange with
    owner bounds / RAW-CHAIN splits (padded elements), counted item by item:
    RAW -- W raw slices of the owner's RAW part from every other rank; CHAIN --
    one partial per hop 0 -> ... -> G-1 and the finished sum into the owner
    unless it is the last rank; w' of every owner range into every other
    replica."""
    G = len(bounds) - 1
    out = inn = 0
    for o in range(G):
        raw, ch, own = split[o] - bounds[o], bounds[o + 1] - split[o], bounds[o + 1] - bounds[o]
        if o == rank:
            inn += W * raw * (G - 1)
            out += own * (G - 1)
        else:
            out += W * raw
            inn += own
        if rank < G - 1:
            out += ch
        if rank > 0:
            inn += ch
        if o != G - 1:
            out += ch if rank == G - 1 else 0
            inn += ch if rank == o else 0
    return 4 * out, 4 * inn


def sched_geometry(key_sizes, chunk_size_bytes: int, G: int, weights, raw_frac):
    """Owner bounds and RAW/CHAIN splits in the padded layout, snapped to chunk
    starts so every chunk has exactly one owner."""
    import bisect
    Ep, offs, _ = capi.phub_plan_ranges(key_sizes, chunk_size_bytes, 1)
    chunks, n = capi.phub_plan_chunks(key_sizes, chunk_size_bytes, 1, capi.PHUB_OWNER_CONTIG)
    starts = sorted(int(offs[chunks[i].key_id]) + int(chunks[i].offset) for i in range(n)) + [Ep]

    def snap(x, lo, hi):
        i = bisect.bisect_left(starts, x)
        cand = [s for s in starts[max(0, i - 1):i + 1] if lo <= s <= hi] or [lo]
        return min(cand, key=lambda s: abs(s - x))

    tot = float(sum(weights))
    bounds, acc = [0], 0.0
    for o in range(G - 1):
        acc += weights[o]
        bounds.append(snap(int(round(Ep * acc / tot)), bounds[-1], Ep))
    bounds.append(Ep)
    split = [snap(bounds[o] + int(round((bounds[o + 1] - bounds[o]) * raw_frac[o])),
                  bounds[o], bounds[o + 1]) for o in range(G)]
    return Ep, bounds, split


class SchedShardedPHub(_DeviceWaitExchange):
    """Scheduled owner-sharded exchange of the N-worker job (
    phub_sched_plan / phub_sched_exchange): per owner range, a RAW part
    exchanged like the push exchange and a CHAIN part summed rank by rank like
    the chained exchange, mixed per SCHED_TABLE so that the busiest NVLink port
    moves the fewest bytes.  One persistent launch per GPU executes this rank's
    item program; every transfer is an NVLink store; the sum is the flat
    worker-order sum (R3), bit-identical to the one-GPU result.  Workers are
    hosted in rank order (rank r: global workers [r*W, (r+1)*W))."""

    def __init__(self, key_sizes, num_workers, chunk_size_bytes=32768, lr=0.1, momentum=0.9,
                 device=None, group=None, block=0, lag=-1, weights=None, raw_frac=None,
                 nslots=2, keep_aggregate=False, consumer_ctas=0, taper=-1, device_barrier=True):
        import torch
        import torch.distributed as dist
        from .phub import PHub, _CudaArray
        self.group = group
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if num_workers % world:
            raise ValueError(f"{num_workers} workers cannot be hosted evenly on {world} ranks")
        self.rank, self.world, self.W = rank, world, num_workers // world
        # measured defaults (profiles/r02_sched5/): G = 2 (the chain plan) 16K-element
        # blocks, no lag; G >= 3 12K-element blocks, chain stages lagging 64 blocks
        self.block = int(block) if block else (16384 if world == 2 else 12288)
        self.lag = int(lag) if lag >= 0 else (0 if world == 2 else 64)
        self.consumer_ctas = int(consumer_ctas)        # 0: auto (phub_sched.consumer_ctas)
        # round barriers inside the launch (phub_sched.device_barrier) instead of two
        # NCCL all-reduces per round
        self.device_barrier = bool(device_barrier)
        # blocks cut 4x finer at each part's ends: 8 at G >= 3 (profiles/r02_sched9/)
        self.taper = int(taper) if taper >= 0 else (0 if world == 2 else 8)
        if weights is None or raw_frac is None:
            if world in SCHED_TABLE:
                weights, raw_frac = SCHED_TABLE[world]
            else:                                      # no table entry: the push exchange
                weights, raw_frac = [1.0 / world] * world, [1.0] * world
        self.shares, self.raw_frac = list(weights), list(raw_frac)     # (weights() is the pull)
        self.device = torch.cuda.current_device() if device is None else int(device)
        dev = self.device
        Ep, self.bounds, self.split = sched_geometry(key_sizes, chunk_size_bytes, world,
                                                     self.shares, self.raw_frac)
        self.hub = PHub(key_sizes, self.W, chunk_size_bytes=chunk_size_bytes, lr=lr,
                        momentum=momentum, rescale=1.0 / num_workers, device=dev,
                        keep_aggregate=keep_aggregate)
        assert self.hub.E_padded == Ep
        items, self.num_flags = capi.phub_sched_plan(world, rank, self.W, self.bounds, self.split,
                                                     self.block, self.lag, self.taper)
        capi.phub_sched_load(self.hub.ctx, world, rank, items, self.num_flags)
        self.nslots = int(nslots)
        self._own = {(sl, k): capi.phub_alloc_shared(dev, 4 * Ep)
                     for sl in range(self.nslots) for k in range(self.W)}
        self._grads = {key: torch.as_tensor(_CudaArray(p, Ep, self), device=f"cuda:{dev}")
                       for key, p in self._own.items()}
        for t in self._grads.values():
            t.zero_()
        raw_len = self.split[rank] - self.bounds[rank]
        self._inbox = capi.phub_alloc_shared(dev, 4 * Ep)
        self._raw = capi.phub_alloc_shared(dev, 4 * world * self.W * max(raw_len, 8))
        self._flags = capi.phub_alloc_shared(dev, 4 * max(self.num_flags, 1))
        torch.as_tensor(_CudaArray(self._flags, max(self.num_flags, 1), self),
                        device=f"cuda:{dev}").zero_()
        h = capi.phub_ipc_get_handle
        mine = (rank, h(dev, self._inbox), h(dev, self._raw), h(dev, self._flags),
                h(dev, self.hub.weights_ptr()))
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        allh.sort(key=lambda x: x[0])
        self._opened = []
        self.inbox, self.raw_inbox, self.flags = [0] * world, [0] * world, [0] * world
        self.inbox[rank], self.raw_inbox[rank], self.flags[rank] = self._inbox, self._raw, self._flags
        reps, err = [], None
        try:
            for q, ih, rh, fh, wh in allh:
                if q == rank:
                    continue
                for hd in (ih, rh, fh, wh):
                    self._opened.append(capi.phub_ipc_open(dev, hd))
                self.inbox[q], self.raw_inbox[q], self.flags[q], pw = self._opened[-4:]
                reps.append(pw)
            capi.phub_set_replicas(self.hub.ctx, reps)
        except capi.PhubError as ex:
            err = ex
        ok = torch.tensor([0 if err else 1], dtype=torch.int32, device=f"cuda:{dev}")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            for p_ in self._opened:
                try:
                    capi.phub_ipc_close(dev, p_)
                except capi.PhubError:
                    pass
            self._grads = {}
            for p_ in list(self._own.values()) + [self._inbox, self._raw, self._flags]:
                capi.phub_free_shared(dev, p_)
            self.hub.close()
            raise PeerMappingError(f"peer mapping failed on some rank ({err or 'other rank'})")
        self.epoch = 0
        self._flag = torch.zeros(1, dtype=torch.float32, device=f"cuda:{dev}")
        self.replica = self.hub.weights()
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)

    @property
    def hosted(self):
        return [self.rank * self.W + k for k in range(self.W)]

    def owned(self):
        """[begin, end) of the padded layout this rank runs Nesterov on."""
        return self.bounds[self.rank], self.bounds[self.rank + 1]

    def gradients(self, slot: int = 0) -> dict:
        return {self.rank * self.W + k: self._grads[(slot, k)] for k in range(self.W)}

    def nvlink_bytes(self):
        """(out, in) bytes of this rank per round under the byte model."""
        return sched_nvlink_bytes(self.bounds, self.split, self.W, self.rank)

    def exchange(self, slot: int = 0):
        """One round in one launch per GPU.  Raises ExchangeFailed if this rank's
        context failed."""
        self._round(lambda: self._exchange(slot))

    def _barriers_per_round(self):
        return 0 if self.device_barrier else 2

    def _exchange(self, slot):
        Ep = self.hub.E_padded
        if not self.device_barrier:
            self.barrier()                   # every replica and inbox free (previous round read)
        for k in range(self.W):
            self.hub.push(k, self._own[(slot, k)], mode="borrow", n=Ep)
        self.epoch += 1
        capi.phub_sched_exchange(self.hub.ctx, self.inbox, self.raw_inbox, self.flags, self.epoch,
                                 self.hub._stream(None), consumer_ctas=self.consumer_ctas,
                                 device_barrier=self.device_barrier)
        if not self.device_barrier:
            self.barrier()                   # every rank's w' stores into this replica are done

    def exchange_host(self, host_grads: dict, host_out: dict, slot: int = 0):
        g = self.gradients(slot)
        for w in self.hosted:
            g[w].copy_(host_grads[w], non_blocking=True)
        self.exchange(slot)
        for w in self.hosted:
            host_out[w].copy_(self.replica, non_blocking=True)

    def weights(self):
        return self.replica

    def close(self):
        import torch
        import torch.distributed as dist
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        capi.phub_set_replicas(self.hub.ctx, [])
        for p in self._opened:
            capi.phub_ipc_close(self.device, p)
        dist.barrier(group=self.group)
        self._grads = {}
        for p in list(self._own.values()) + [self._inbox, self._raw, self._flags]:
            capi.phub_free_shared(self.device, p)
        self._own = {}
        self.hub.close()
