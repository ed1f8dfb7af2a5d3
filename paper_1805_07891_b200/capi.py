"""ctypes binding of include/phub.h -- argument marshalling only.

Every function here has the name of the C entry point it calls and does no
computation of its own: each step of the hot path runs in libphub.so's sm_100a
kernels.  There is no fallback: if libphub.so is missing or fails to load,
importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libphub.so")

# ----------------------------------------------------------------- constants
PHUB_OK = 0
STATUS_NAMES = [
    "PHUB_OK", "PHUB_ERR_INVALID_ARGUMENT", "PHUB_ERR_INVALID_MANIFEST",
    "PHUB_ERR_INVALID_CHUNK_SIZE", "PHUB_ERR_INVALID_INIT", "PHUB_ERR_BAD_WORKER",
    "PHUB_ERR_BAD_KEY", "PHUB_ERR_LENGTH_MISMATCH", "PHUB_ERR_DUPLICATE_PUSH",
    "PHUB_ERR_INCOMPLETE", "PHUB_ERR_CUDA", "PHUB_ERR_OUT_OF_MEMORY", "PHUB_ERR_UNSUPPORTED",
    "PHUB_ERR_SYNC_TIMEOUT",
]
for _i, _n in enumerate(STATUS_NAMES):
    globals()[_n] = _i
PHUB_ALL_KEYS = -1
PHUB_OWNED_RANGE = -2
PHUB_COPY, PHUB_BORROW = 0, 1
PHUB_OWNER_LPT, PHUB_OWNER_CONTIG = 0, 1
PHUB_OPT_KERNEL, PHUB_OPT_GRID, PHUB_OPT_TILE_ELEMS, PHUB_OPT_CACHE = 1, 2, 3, 4
PHUB_OPT_FLAT_ONESHOT, PHUB_OPT_L2_RESIDENT, PHUB_OPT_SCHED_TRACE = 7, 8, 9
PHUB_CROSS_RACK_SHARDED, PHUB_CROSS_RACK_RING = 0, 1
(PHUB_KERNEL_AUTO, PHUB_KERNEL_FLAT, PHUB_KERNEL_TILES, PHUB_KERNEL_FLAT128,
 PHUB_KERNEL_WIDE, PHUB_KERNEL_BULK) = range(6)
PHUB_CACHE_ENABLED, PHUB_CACHE_BYPASS, PHUB_CACHE_RESIDENT = 0, 1, 2
(PHUB_ITEM_RAW_PUSH, PHUB_ITEM_CHAIN, PHUB_ITEM_CONSUME_RAW,
 PHUB_ITEM_CONSUME_FINAL) = 1, 2, 3, 4
PHUB_NO_FLAG = 0xFFFFFFFF


class phub_chunk(C.Structure):
    _fields_ = [("vkey_id", C.c_uint32), ("key_id", C.c_uint32), ("offset", C.c_uint64),
                ("length", C.c_uint64), ("owner", C.c_int32), ("reserved", C.c_int32)]


class phub_sync(C.Structure):
    _fields_ = [("wait_flag", C.c_void_p), ("wait_value", C.c_uint32),
                ("signal_flag", C.c_void_p), ("signal_value", C.c_uint32),
                ("block_elems", C.c_uint64)]


class phub_hier(C.Structure):
    _fields_ = [("num_racks", C.c_int32), ("block_elems", C.c_uint64),
                ("inbox", C.POINTER(C.c_void_p)), ("peer_inbox", C.POINTER(C.c_void_p)),
                ("flags", C.c_void_p), ("peer_flags", C.POINTER(C.c_void_p)),
                ("epoch", C.c_uint32), ("worker_order", C.c_int32),
                ("device_barrier", C.c_int32)]


class phub_sched_item(C.Structure):
    _fields_ = [("lo", C.c_uint64), ("hi", C.c_uint64), ("base", C.c_uint64), ("len", C.c_uint64),
                ("type", C.c_uint32), ("dst", C.c_int32), ("wait_flag", C.c_uint32),
                ("signal_flag", C.c_uint32)]


class phub_sched(C.Structure):
    _fields_ = [("inbox", C.POINTER(C.c_void_p)), ("raw_inbox", C.POINTER(C.c_void_p)),
                ("flags", C.POINTER(C.c_void_p)), ("epoch", C.c_uint32),
                ("consumer_ctas", C.c_int32), ("device_barrier", C.c_int32)]


class phub_config(C.Structure):
    _fields_ = [
        ("key_num_elements", C.POINTER(C.c_uint64)),
        ("num_keys", C.c_int32),
        ("num_workers", C.c_int32),
        ("chunk_size_bytes", C.c_uint64),
        ("lr", C.c_float),
        ("momentum", C.c_float),
        ("rescale", C.c_float),
        ("device", C.c_int32),
        ("num_owners", C.c_int32),
        ("owner_rank", C.c_int32),
        ("owner_policy", C.c_int32),
        ("keep_aggregate", C.c_int32),
        ("init_weights", C.c_void_p),
        ("init_num_elements", C.c_uint64),
    ]


phub_ctx = C.c_void_p
_u64p = C.POINTER(C.c_uint64)

_SIGS = {
    "phub_config_default": (None, [C.POINTER(phub_config)]),
    "phub_init": (C.c_int, [C.POINTER(phub_config), C.POINTER(phub_ctx)]),
    "phub_destroy": (C.c_int, [phub_ctx]),
    "phub_push": (C.c_int, [phub_ctx, C.c_int32, C.c_int32, C.c_void_p, C.c_uint64, C.c_int32,
                            C.c_void_p]),
    "phub_aggregate_optimize": (C.c_int, [phub_ctx, C.c_void_p]),
    "phub_push_batch": (C.c_int, [phub_ctx, C.c_int32, C.POINTER(C.c_int32),
                                  C.POINTER(C.c_int32), C.POINTER(C.c_void_p), _u64p, C.c_int32,
                                  C.c_void_p, C.POINTER(C.c_int32)]),
    "phub_aggregate_ready": (C.c_int, [phub_ctx, C.c_void_p, _u64p]),
    "phub_aggregate_range": (C.c_int, [phub_ctx, C.c_uint64, C.c_uint64, C.c_void_p,
                                       C.c_void_p]),
    "phub_partial_sum": (C.c_int, [phub_ctx, C.POINTER(C.c_void_p), C.c_int32, C.c_void_p,
                                   C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p]),
    "phub_sync_timeouts": (C.c_int, [phub_ctx, C.POINTER(C.c_uint32)]),
    "phub_synchronize": (C.c_int, [phub_ctx, C.c_void_p]),
    "phub_check": (C.c_int, [phub_ctx]),
    "phub_hier_beneficial": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double,
                                       C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]),
    "phub_pull": (C.c_int, [phub_ctx, C.c_int32, C.c_void_p, C.c_uint64, C.c_void_p]),
    "phub_pushpull": (C.c_int, [phub_ctx, C.c_int32, C.c_void_p, C.c_uint64, C.c_int32,
                                C.c_void_p, C.c_void_p]),
    "phub_weights": (C.c_int, [phub_ctx, C.POINTER(C.c_void_p)]),
    "phub_layout": (C.c_int, [phub_ctx, _u64p, _u64p, _u64p]),
    "phub_num_chunks": (C.c_int, [phub_ctx, _u64p]),
    "phub_chunk_table": (C.c_int, [phub_ctx, C.POINTER(phub_chunk), C.c_uint64]),
    "phub_plan_chunks": (C.c_int, [_u64p, C.c_int32, C.c_uint64, C.c_int32, C.c_int32,
                                   C.POINTER(phub_chunk), C.c_uint64, _u64p]),
    "phub_plan_ranges": (C.c_int, [_u64p, C.c_int32, C.c_uint64, C.c_int32, _u64p, _u64p, _u64p,
                                   _u64p]),
    "phub_owner_range": (C.c_int, [phub_ctx, C.c_int32, _u64p, _u64p]),
    "phub_owned_elements": (C.c_int, [phub_ctx, _u64p]),
    "phub_load_state": (C.c_int, [phub_ctx, C.c_void_p, C.c_void_p]),
    "phub_read_state": (C.c_int, [phub_ctx, C.c_void_p, C.c_void_p, C.c_void_p]),
    "phub_iteration": (C.c_int, [phub_ctx, _u64p]),
    "phub_kernel_launches": (C.c_int, [phub_ctx, _u64p]),
    "phub_set_option": (C.c_int, [phub_ctx, C.c_int32, C.c_int64]),
    "phub_set_replicas": (C.c_int, [phub_ctx, C.POINTER(C.c_void_p), C.c_int32]),
    "phub_hier_exchange": (C.c_int, [phub_ctx, C.c_void_p, C.c_void_p]),
    "phub_sched_plan": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, _u64p, _u64p, C.c_uint64,
                                  C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64, _u64p,
                                  C.POINTER(C.c_uint32)]),
    "phub_sched_load": (C.c_int, [phub_ctx, C.c_int32, C.c_int32, C.c_void_p, C.c_uint64,
                                  C.c_uint32]),
    "phub_sched_exchange": (C.c_int, [phub_ctx, C.c_void_p, C.c_void_p]),
    "phub_alloc_shared": (C.c_int, [C.c_int32, C.c_uint64, C.POINTER(C.c_void_p)]),
    "phub_free_shared": (C.c_int, [C.c_int32, C.c_void_p]),
    "phub_ipc_get_handle": (C.c_int, [C.c_int32, C.c_void_p, C.c_void_p]),
    "phub_ipc_open": (C.c_int, [C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)]),
    "phub_ipc_close": (C.c_int, [C.c_int32, C.c_void_p]),
    "phub_status_string": (C.c_char_p, [C.c_int]),
    "phub_last_error": (C.c_char_p, [phub_ctx]),
}
EXPORTS = tuple(_SIGS)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_1805_07891_b200/build.py` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()


class PhubError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{where}: {name}" + (f" ({detail})" if detail else ""))


def _check(st: int, where: str, ctx=None):
    if st != PHUB_OK:
        d = _lib.phub_last_error(ctx)          # ctx None -> this thread's init error
        raise PhubError(st, where, d.decode() if d else "")


# ------------------------------------------------- same-named thin wrappers
def phub_config_default() -> phub_config:
    cfg = phub_config()
    _lib.phub_config_default(C.byref(cfg))
    return cfg


def phub_init(cfg: phub_config):
    ctx = phub_ctx()
    _check(_lib.phub_init(C.byref(cfg), C.byref(ctx)), "phub_init")
    return ctx


def phub_destroy(ctx):
    _check(_lib.phub_destroy(ctx), "phub_destroy")


def phub_push(ctx, worker: int, key: int, grad_ptr: int, n: int, mode: int, stream: int = 0):
    _check(_lib.phub_push(ctx, worker, key, grad_ptr, n, mode, stream), "phub_push", ctx)


def phub_push_batch(ctx, workers, keys, ptrs, lens, mode: int, stream: int = 0) -> None:
    n = len(workers)
    wa = (C.c_int32 * max(n, 1))(*workers)
    ka = (C.c_int32 * max(n, 1))(*keys)
    pa = (C.c_void_p * max(n, 1))(*ptrs)
    la = (C.c_uint64 * max(n, 1))(*lens)
    bad = C.c_int32(-1)
    st = _lib.phub_push_batch(ctx, n, wa, ka, pa, la, mode, stream, C.byref(bad))
    if st != PHUB_OK:
        d = _lib.phub_last_error(ctx)
        raise PhubError(st, f"phub_push_batch[{bad.value}]", d.decode() if d else "")


def phub_aggregate_optimize(ctx, stream: int = 0):
    _check(_lib.phub_aggregate_optimize(ctx, stream), "phub_aggregate_optimize", ctx)


def phub_aggregate_ready(ctx, stream: int = 0) -> int:
    n = C.c_uint64()
    _check(_lib.phub_aggregate_ready(ctx, stream, C.byref(n)), "phub_aggregate_ready", ctx)
    return int(n.value)


def _sync(wait=None, signal=None, block=0):
    """phub_sync from (flag_ptr, value) pairs; None when nothing is given.
    block > 0: the flag pointers are per-block arrays (block-streaming form)."""
    if wait is None and signal is None:
        return None
    s = phub_sync()
    if wait is not None:
        s.wait_flag, s.wait_value = wait
    if signal is not None:
        s.signal_flag, s.signal_value = signal
    s.block_elems = int(block)
    return C.byref(s)


def phub_aggregate_range(ctx, begin: int, end: int, stream: int = 0, wait=None, signal=None,
                         block: int = 0):
    _check(_lib.phub_aggregate_range(ctx, begin, end, _sync(wait, signal, block), stream),
           "phub_aggregate_range", ctx)


def phub_partial_sum(ctx, srcs, dst: int, begin: int, end: int, stream: int = 0, wait=None,
                     signal=None, block: int = 0):
    arr = (C.c_void_p * max(len(srcs), 1))(*srcs)
    _check(_lib.phub_partial_sum(ctx, arr, len(srcs), dst, begin, end,
                                 _sync(wait, signal, block), stream), "phub_partial_sum", ctx)


def phub_sync_timeouts(ctx) -> int:
    n = C.c_uint32()
    _check(_lib.phub_sync_timeouts(ctx, C.byref(n)), "phub_sync_timeouts", ctx)
    return int(n.value)


def phub_check(ctx) -> int:
    """The context's status without synchronizing (0 = PHUB_OK; never raises)."""
    return int(_lib.phub_check(ctx))


def phub_synchronize(ctx, stream: int = 0):
    _check(_lib.phub_synchronize(ctx, stream), "phub_synchronize", ctx)


def phub_hier_beneficial(workers_per_rack: int, racks: int, b_pbox: float, b_wkr: float,
                         b_core: float, cross_rack: int = PHUB_CROSS_RACK_SHARDED):
    """(beneficial, lhs, rhs) of the P:760-763 model (host-only)."""
    ben, lhs, rhs = C.c_int32(), C.c_double(), C.c_double()
    _check(_lib.phub_hier_beneficial(workers_per_rack, racks, b_pbox, b_wkr, b_core, cross_rack,
                                     C.byref(ben), C.byref(lhs), C.byref(rhs)),
           "phub_hier_beneficial", None)
    return bool(ben.value), float(lhs.value), float(rhs.value)


def phub_pull(ctx, key: int, dst_ptr: int, n: int, stream: int = 0):
    _check(_lib.phub_pull(ctx, key, dst_ptr, n, stream), "phub_pull", ctx)


def phub_pushpull(ctx, worker: int, grad_ptr: int, n: int, mode: int, dst_ptr, stream: int = 0):
    _check(_lib.phub_pushpull(ctx, worker, grad_ptr, n, mode, dst_ptr, stream), "phub_pushpull",
           ctx)


def phub_weights(ctx) -> int:
    p = C.c_void_p()
    _check(_lib.phub_weights(ctx, C.byref(p)), "phub_weights", ctx)
    return int(p.value or 0)


def phub_layout(ctx, num_keys: int):
    E, Ep = C.c_uint64(), C.c_uint64()
    offs = (C.c_uint64 * num_keys)()
    _check(_lib.phub_layout(ctx, C.byref(E), C.byref(Ep), offs), "phub_layout", ctx)
    return int(E.value), int(Ep.value), list(offs)


def phub_num_chunks(ctx) -> int:
    n = C.c_uint64()
    _check(_lib.phub_num_chunks(ctx, C.byref(n)), "phub_num_chunks", ctx)
    return int(n.value)


def phub_chunk_table(ctx):
    n = phub_num_chunks(ctx)
    arr = (phub_chunk * max(n, 1))()
    _check(_lib.phub_chunk_table(ctx, arr, n), "phub_chunk_table", ctx)
    return arr, n


def phub_plan_chunks(key_sizes, chunk_size_bytes: int, num_owners: int, owner_policy: int):
    """Host-only chunk table (no device): list-of-structs array and count."""
    n = (C.c_uint64 * max(len(key_sizes), 1))(*[int(x) for x in key_sizes])
    cnt = C.c_uint64()
    _check(_lib.phub_plan_chunks(n, len(key_sizes), chunk_size_bytes, num_owners, owner_policy,
                                 None, 0, C.byref(cnt)), "phub_plan_chunks", None)
    arr = (phub_chunk * max(cnt.value, 1))()
    _check(_lib.phub_plan_chunks(n, len(key_sizes), chunk_size_bytes, num_owners, owner_policy,
                                 arr, cnt.value, C.byref(cnt)), "phub_plan_chunks", None)
    return arr, int(cnt.value)


def phub_plan_ranges(key_sizes, chunk_size_bytes: int, num_owners: int):
    """Host-only: (E_padded, key_offsets, [(begin, end) per owner]) under CONTIG."""
    K = len(key_sizes)
    n = (C.c_uint64 * max(K, 1))(*[int(x) for x in key_sizes])
    Ep = C.c_uint64()
    offs = (C.c_uint64 * max(K, 1))()
    b = (C.c_uint64 * num_owners)()
    e = (C.c_uint64 * num_owners)()
    _check(_lib.phub_plan_ranges(n, K, chunk_size_bytes, num_owners, C.byref(Ep), offs, b, e),
           "phub_plan_ranges", None)
    return int(Ep.value), list(offs)[:K], list(zip(list(b), list(e)))


def phub_owner_range(ctx, owner: int):
    b, e = C.c_uint64(), C.c_uint64()
    _check(_lib.phub_owner_range(ctx, owner, C.byref(b), C.byref(e)), "phub_owner_range", ctx)
    return int(b.value), int(e.value)


def phub_owned_elements(ctx) -> int:
    n = C.c_uint64()
    _check(_lib.phub_owned_elements(ctx, C.byref(n)), "phub_owned_elements", ctx)
    return int(n.value)


def phub_load_state(ctx, w_ptr, v_ptr):
    _check(_lib.phub_load_state(ctx, w_ptr, v_ptr), "phub_load_state", ctx)


def phub_read_state(ctx, w_ptr, v_ptr, agg_ptr):
    _check(_lib.phub_read_state(ctx, w_ptr, v_ptr, agg_ptr), "phub_read_state", ctx)


def phub_iteration(ctx) -> int:
    n = C.c_uint64()
    _check(_lib.phub_iteration(ctx, C.byref(n)), "phub_iteration", ctx)
    return int(n.value)


def phub_kernel_launches(ctx) -> int:
    n = C.c_uint64()
    _check(_lib.phub_kernel_launches(ctx, C.byref(n)), "phub_kernel_launches", ctx)
    return int(n.value)


def phub_set_option(ctx, option: int, value: int):
    _check(_lib.phub_set_option(ctx, option, value), "phub_set_option", ctx)


def phub_set_replicas(ctx, ptrs):
    arr = (C.c_void_p * max(len(ptrs), 1))(*ptrs)
    _check(_lib.phub_set_replicas(ctx, arr, len(ptrs)), "phub_set_replicas", ctx)


def phub_hier_exchange(ctx, num_racks: int, block: int, inbox, peer_inbox, flags: int,
                       peer_flags, epoch: int, stream: int = 0, worker_order: bool = False,
                       device_barrier: bool = False):
    """Hierarchical reduction round (phub.h phub_hier_exchange); pointer lists
    have num_racks entries (this rack's entry ignored, may be 0)."""
    R = int(num_racks)
    def arr(xs):
        return (C.c_void_p * max(R, 1))(*[int(x or 0) for x in xs]) if xs else None
    ib, pib, pf = arr(inbox), arr(peer_inbox), arr(peer_flags)     # alive across the call
    h = phub_hier(R, int(block), ib, pib, flags or None, pf, int(epoch), int(bool(worker_order)),
                  int(bool(device_barrier)))
    _check(_lib.phub_hier_exchange(ctx, C.byref(h), stream), "phub_hier_exchange", ctx)


def phub_sched_plan(ranks: int, rank: int, workers_per_rank: int, bounds, split,
                    block_elems: int, lag_blocks: int = 0, taper_blocks: int = 0):
    """Item program of `rank` (phub.h phub_sched_plan): (items array, num_flags)."""
    b = (C.c_uint64 * len(bounds))(*[int(x) for x in bounds])
    sp = (C.c_uint64 * len(split))(*[int(x) for x in split])
    n, nf = C.c_uint64(), C.c_uint32()
    args = (ranks, rank, workers_per_rank, b, sp, int(block_elems), int(lag_blocks),
            int(taper_blocks))
    _check(_lib.phub_sched_plan(*args, None, 0, C.byref(n), C.byref(nf)), "phub_sched_plan", None)
    items = (phub_sched_item * n.value)()
    _check(_lib.phub_sched_plan(*args, items, n.value, C.byref(n), C.byref(nf)),
           "phub_sched_plan", None)
    return items, nf.value


def phub_sched_load(ctx, ranks: int, rank: int, items, num_flags: int):
    _check(_lib.phub_sched_load(ctx, ranks, rank, items, len(items), num_flags),
           "phub_sched_load", ctx)


def phub_sched_exchange(ctx, inbox, raw_inbox, flags, epoch: int, stream: int = 0,
                        consumer_ctas: int = 0, device_barrier: bool = False):
    """One scheduled round (phub.h phub_sched_exchange); pointer lists per rank."""
    R = len(inbox)
    arr = lambda xs: (C.c_void_p * R)(*[x or None for x in xs])  # noqa: E731
    s = phub_sched(arr(inbox), arr(raw_inbox), arr(flags), int(epoch), int(consumer_ctas),
                   int(bool(device_barrier)))
    _check(_lib.phub_sched_exchange(ctx, C.byref(s), stream), "phub_sched_exchange", ctx)


def phub_alloc_shared(device: int, nbytes: int) -> int:
    p = C.c_void_p()
    _check(_lib.phub_alloc_shared(device, nbytes, C.byref(p)), "phub_alloc_shared", None)
    return int(p.value)


def phub_free_shared(device: int, ptr: int):
    _check(_lib.phub_free_shared(device, ptr), "phub_free_shared", None)


def phub_ipc_get_handle(device: int, ptr: int) -> bytes:
    buf = C.create_string_buffer(64)
    _check(_lib.phub_ipc_get_handle(device, ptr, buf), "phub_ipc_get_handle", None)
    return buf.raw


def phub_ipc_open(device: int, handle: bytes) -> int:
    p = C.c_void_p()
    buf = C.create_string_buffer(bytes(handle), 64)
    _check(_lib.phub_ipc_open(device, buf, C.byref(p)), "phub_ipc_open", None)
    return int(p.value)


def phub_ipc_close(device: int, ptr: int):
    _check(_lib.phub_ipc_close(device, ptr), "phub_ipc_close", None)


def phub_status_string(st: int) -> str:
    return _lib.phub_status_string(st).decode()


def phub_last_error(ctx) -> str:
    r = _lib.phub_last_error(ctx)
    return r.decode() if r else ""


def raw_lib():
    """The loaded ctypes library (tests check the exported symbols)."""
    return _lib
