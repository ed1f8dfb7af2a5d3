"""Pythonic handle over the C ABI -- marshalling only (no computation).

    hub = PHub(key_sizes, num_workers=8)                  # phub_init
    for w in range(8):
        hub.push(w, grads[w])                             # phub_push (BORROW, zero copy)
    hub.aggregate_optimize()                              # one fused sm_100a kernel
    w_new = hub.weights()                                 # zero-copy pull (torch view)

Buffers may be torch tensors (device or host), numpy arrays (host) or raw
pointers with an explicit length.  Streams default to torch's current stream
on the context's device so CUDA events recorded by torch bracket the work.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi
from .capi import PHUB_ALL_KEYS, PHUB_BORROW, PHUB_COPY

_MODES = {"borrow": PHUB_BORROW, "copy": PHUB_COPY, PHUB_BORROW: PHUB_BORROW, PHUB_COPY: PHUB_COPY}
_POLICIES = {"lpt": capi.PHUB_OWNER_LPT, "contig": capi.PHUB_OWNER_CONTIG,
             capi.PHUB_OWNER_LPT: capi.PHUB_OWNER_LPT, capi.PHUB_OWNER_CONTIG: capi.PHUB_OWNER_CONTIG}


def _ptr_len(buf, n=None):
    """(pointer, element count) of a float32 buffer; no data is touched."""
    if isinstance(buf, int):
        if n is None:
            raise ValueError("raw pointer needs an explicit length")
        return buf, int(n)
    if isinstance(buf, np.ndarray):
        if buf.dtype != np.float32 or not buf.flags["C_CONTIGUOUS"]:
            raise ValueError("numpy buffer must be C-contiguous float32")
        return buf.ctypes.data, buf.size
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(buf, torch.Tensor):
        if buf.dtype != torch.float32 or not buf.is_contiguous():
            raise ValueError("tensor must be contiguous float32")
        return buf.data_ptr(), buf.numel()
    raise TypeError(f"unsupported buffer type {type(buf)}")


class _CudaArray:
    """__cuda_array_interface__ view of a device range owned by a context."""

    def __init__(self, ptr, n, owner):
        self._owner = owner
        self.__cuda_array_interface__ = {
            "shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3,
            "strides": None, "stream": None,
        }


class PHub:
    def __init__(self, key_sizes, num_workers, chunk_size_bytes=32768, lr=0.1, momentum=0.9,
                 rescale=0.0, device=0, num_owners=1, owner_rank=0, owner_policy="contig",
                 keep_aggregate=False, init_weights=None):
        self.key_sizes = [int(x) for x in key_sizes]
        self._sizes = (C.c_uint64 * max(len(self.key_sizes), 1))(*self.key_sizes)
        cfg = capi.phub_config_default()
        cfg.key_num_elements = self._sizes
        cfg.num_keys = len(self.key_sizes)
        cfg.num_workers = int(num_workers)
        cfg.chunk_size_bytes = int(chunk_size_bytes)
        cfg.lr = float(lr)
        cfg.momentum = float(momentum)
        cfg.rescale = float(rescale)
        cfg.device = int(device)
        cfg.num_owners = int(num_owners)
        cfg.owner_rank = int(owner_rank)
        cfg.owner_policy = _POLICIES[owner_policy]
        cfg.keep_aggregate = int(bool(keep_aggregate))
        if init_weights is not None:
            p, n = _ptr_len(init_weights)
            cfg.init_weights = p
            cfg.init_num_elements = n
        self.device = int(device)
        self.num_workers = int(num_workers)
        self.num_owners = int(num_owners)
        self.owner_rank = int(owner_rank)
        self.keep_aggregate = bool(keep_aggregate)
        self.ctx = capi.phub_init(cfg)
        self.E, self.E_padded, self.key_offsets = capi.phub_layout(self.ctx, len(self.key_sizes))

    # -------------------------------------------------------------- streams
    def _stream(self, stream):
        if stream is None:
            try:
                import torch
                if torch.cuda.is_available():
                    return torch.cuda.current_stream(self.device).cuda_stream
            except ImportError:  # pragma: no cover
                pass
            return 0
        if isinstance(stream, int):
            return stream
        return stream.cuda_stream

    # ------------------------------------------------------------- hot path
    def push(self, worker, grad, key=PHUB_ALL_KEYS, mode="borrow", n=None, stream=None):
        p, cnt = _ptr_len(grad, n)
        capi.phub_push(self.ctx, int(worker), int(key), p, cnt, _MODES[mode], self._stream(stream))

    def push_batch(self, entries, mode="borrow", stream=None):
        """entries: iterable of (worker, key, buffer) -- one C call, all-or-nothing."""
        ws, ks, ps, ls = [], [], [], []
        for w, k, buf in entries:
            p, n = _ptr_len(buf)
            ws.append(int(w))
            ks.append(int(k))
            ps.append(p)
            ls.append(n)
        capi.phub_push_batch(self.ctx, ws, ks, ps, ls, _MODES[mode], self._stream(stream))

    def aggregate_optimize(self, stream=None):
        capi.phub_aggregate_optimize(self.ctx, self._stream(stream))

    def aggregate_ready(self, stream=None) -> int:
        """Streaming: aggregate every fully-pushed key not yet aggregated."""
        return capi.phub_aggregate_ready(self.ctx, self._stream(stream))

    def pull(self, dst, key=PHUB_ALL_KEYS, n=None, stream=None):
        p, cnt = _ptr_len(dst, n)
        capi.phub_pull(self.ctx, int(key), p, cnt, self._stream(stream))

    def pushpull(self, worker, grad, dst=None, mode="borrow", stream=None):
        p, cnt = _ptr_len(grad)
        d = _ptr_len(dst)[0] if dst is not None else None
        capi.phub_pushpull(self.ctx, int(worker), p, cnt, _MODES[mode], d, self._stream(stream))

    def weights_ptr(self) -> int:
        return capi.phub_weights(self.ctx)

    def weights(self):
        """Zero-copy pull: torch view of the padded weight replica on the device."""
        import torch
        return torch.as_tensor(_CudaArray(self.weights_ptr(), self.E_padded, self),
                               device=f"cuda:{self.device}")

    # ---------------------------------------------------------- introspection
    def chunk_table(self) -> dict:
        arr, n = capi.phub_chunk_table(self.ctx)
        a = np.ctypeslib.as_array(arr)[:n]
        return {f: np.array(a[f]) for f in ("vkey_id", "key_id", "offset", "length", "owner")}

    def owner_range(self, owner=None):
        return capi.phub_owner_range(self.ctx, self.owner_rank if owner is None else int(owner))

    def owned_elements(self) -> int:
        return capi.phub_owned_elements(self.ctx)

    def read_state(self):
        """(w, v, s) as E-element key-major numpy arrays (s None unless keep_aggregate)."""
        w = np.empty(self.E, np.float32)
        v = np.empty(self.E, np.float32)
        s = np.empty(self.E, np.float32) if self.keep_aggregate else None
        capi.phub_read_state(self.ctx, w.ctypes.data, v.ctypes.data,
                             s.ctypes.data if s is not None else None)
        return w, v, s

    def load_state(self, w=None, v=None):
        pw = _ptr_len(w)[0] if w is not None else None
        pv = _ptr_len(v)[0] if v is not None else None
        for buf in (w, v):
            if buf is not None and _ptr_len(buf)[1] != self.E:
                raise ValueError("state arrays must have E elements")
        capi.phub_load_state(self.ctx, pw, pv)

    def synchronize(self, stream=None):
        """Wait for this context's work; raises PhubError(PHUB_ERR_SYNC_TIMEOUT) if a
        device-side wait expired (the round is then incomplete)."""
        capi.phub_synchronize(self.ctx, self._stream(stream) if stream is not None else 0)

    def set_option(self, option, value):
        capi.phub_set_option(self.ctx, int(option), int(value))

    @property
    def iteration(self) -> int:
        return capi.phub_iteration(self.ctx)

    @property
    def kernel_launches(self) -> int:
        return capi.phub_kernel_launches(self.ctx)

    def padded_index(self):
        """Index array mapping real element i -> its padded-layout offset."""
        idx = np.empty(self.E, np.int64)
        s = 0
        for k, nk in enumerate(self.key_sizes):
            idx[s:s + nk] = self.key_offsets[k] + np.arange(nk)
            s += nk
        return idx

    def close(self):
        if getattr(self, "ctx", None):
            capi.phub_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
