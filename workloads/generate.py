"""Counter-based synthetic value generator (splitmix64), host and device.

Every value is a pure function of (stream, index), so the oracle side and the
CUDA side can each materialise exactly the same fp32 inputs -- whole arrays for
small configs, or single sampled elements for the full-size configs -- without
moving gigabytes between them.  Nothing here computes any part of the PHub
method; it is input synthesis only.

Value recipe (all exactly representable in fp32, so numpy and torch agree
bit for bit):

    z       = splitmix64(stream_key(stream) + index)         (uint64, wrapping)
    isum    = sum of the four 16-bit fields of z              (0 .. 262140)
    value   = (isum - 131070) * 2**-shift                     (Irwin-Hall(4) ~ normal)

The std of (isum - 131070) is ~2**15.21, so ``shift=25`` gives gradients with
std ~2**-10 (SURVEY.md 8(d) "g ~ 2^-10 N(0,1)"), ``shift=20`` weights with
std ~0.036.

Those values carry at most 17 significant bits at one fixed scale, so any sum
of <= 128 of them is exact in fp32 in ANY order: they cannot tell a
worker-order sum from a reversed or tree-ordered one.  The parity tests
therefore use the *full-mantissa* recipe (``fullmant_*``), built bit by bit:

    bits  = sign << 31 | (127 - e) << 23 | mantissa23
    sign  = bit 63 of z,  e = (z >> 23) % 31,  mantissa23 = z & 0x7FFFFF

i.e. a random 24-bit significand with a random binade 2^-e, e in [0, 30]
(magnitudes in [2^-30, 2)), random sign.  Nearly every fp32 addition of two
such values rounds, so summing the same workers in another order changes the
result on most elements (tests/test_generate.py pins this).  Integer
construction only: numpy and torch produce identical bits.
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 1805_07891
GRAD_SHIFT = 25
WEIGHT_SHIFT = 20
MOMENTUM_SHIFT = 25

_M64 = (1 << 64) - 1
_C0 = 0x9E3779B97F4A7C15
_C1 = 0xBF58476D1CE4E5B9
_C2 = 0x94D049BB133111EB


def _splitmix64_int(x: int) -> int:
    z = (x + _C0) & _M64
    z = ((z ^ (z >> 30)) * _C1) & _M64
    z = ((z ^ (z >> 27)) * _C2) & _M64
    return z ^ (z >> 31)


def stream_key(stream: int) -> int:
    return _splitmix64_int((BASE_SEED << 20) ^ (stream & 0xFFFFF))


def grad_stream(worker: int) -> int:
    """Stream id of worker ``worker``'s gradient (one stream per worker)."""
    return 1000 + worker


def weight_stream() -> int:
    return 1


def momentum_stream() -> int:
    return 2


# ---------------------------------------------------------------- numpy (host)
def _splitmix64_np(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(_C0)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_C1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_C2)
        return z ^ (z >> np.uint64(31))


def _fields_sum_np(z: np.ndarray) -> np.ndarray:
    m = np.uint64(0xFFFF)
    s = (z & m) + ((z >> np.uint64(16)) & m) + ((z >> np.uint64(32)) & m) + (z >> np.uint64(48))
    return s.astype(np.int64)


def values_at_np(stream: int, index: np.ndarray, shift: int) -> np.ndarray:
    """fp32 values of ``stream`` at arbitrary element indices."""
    idx = np.asarray(index, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = _splitmix64_np(idx + np.uint64(stream_key(stream)))
    isum = _fields_sum_np(z) - 131070
    return (isum.astype(np.float32) * np.float32(2.0 ** -shift)).astype(np.float32)


def values_np(stream: int, start: int, count: int, shift: int) -> np.ndarray:
    """fp32 values of ``stream`` at indices start .. start+count-1."""
    return values_at_np(stream, np.arange(start, start + count, dtype=np.uint64), shift)


def dyadic_np(stream: int, count: int, start: int = 0) -> np.ndarray:
    """Dyadic values k/256 with |k| <= 1023: any N<=64 of them sum exactly in fp32."""
    with np.errstate(over="ignore"):
        z = _splitmix64_np(np.arange(start, start + count, dtype=np.uint64)
                           + np.uint64(stream_key(stream)))
    k = (z % np.uint64(2047)).astype(np.int64) - 1023
    return (k.astype(np.float32) / np.float32(256.0)).astype(np.float32)


FULLMANT_BINADES = 31          # e in [0, 30]: magnitudes in [2^-30, 2)


def _fullmant_bits_np(z: np.ndarray) -> np.ndarray:
    sign = (z >> np.uint64(63)) << np.uint64(31)
    e = (z >> np.uint64(23)) % np.uint64(FULLMANT_BINADES)
    bits = sign | ((np.uint64(127) - e) << np.uint64(23)) | (z & np.uint64(0x7FFFFF))
    return bits.astype(np.uint32)


def fullmant_at_np(stream: int, index: np.ndarray) -> np.ndarray:
    """Full-mantissa fp32 values of ``stream`` at arbitrary element indices."""
    idx = np.asarray(index, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = _splitmix64_np(idx + np.uint64(stream_key(stream)))
    return _fullmant_bits_np(z).view(np.float32)


def fullmant_np(stream: int, start: int, count: int) -> np.ndarray:
    """Full-mantissa fp32 values of ``stream`` at indices start .. start+count-1."""
    return fullmant_at_np(stream, np.arange(start, start + count, dtype=np.uint64))


# ------------------------------------------------------------- torch (device)
def _s64(c: int) -> int:
    return c - (1 << 64) if c >= (1 << 63) else c


def _lsr(t, s: int):
    import torch  # noqa: F401
    return (t >> s) & ((1 << (64 - s)) - 1)


def _splitmix64_torch(x):
    z = x + _s64(_C0)
    z = (z ^ _lsr(z, 30)) * _s64(_C1)
    z = (z ^ _lsr(z, 27)) * _s64(_C2)
    return z ^ _lsr(z, 31)


def values_torch(stream: int, start: int, count: int, shift: int, device, out=None,
                 block: int = 1 << 25):
    """Same values as :func:`values_np`, generated on ``device`` (blocked)."""
    import torch
    if out is None:
        out = torch.empty(count, dtype=torch.float32, device=device)
    key = _s64(stream_key(stream))
    scale = 2.0 ** -shift
    for b in range(0, count, block):
        n = min(block, count - b)
        idx = torch.arange(start + b, start + b + n, dtype=torch.int64, device=device)
        z = _splitmix64_torch(idx + key)
        isum = (z & 0xFFFF) + ((z >> 16) & 0xFFFF) + ((z >> 32) & 0xFFFF) + ((z >> 48) & 0xFFFF)
        out[b:b + n] = (isum - 131070).to(torch.float32) * scale
    return out


def fullmant_torch(stream: int, start: int, count: int, device, out=None, block: int = 1 << 25):
    """Same values as :func:`fullmant_np`, generated on ``device`` (blocked)."""
    import torch
    if out is None:
        out = torch.empty(count, dtype=torch.float32, device=device)
    key = _s64(stream_key(stream))
    ov = out.view(torch.int32)
    for b in range(0, count, block):
        n = min(block, count - b)
        idx = torch.arange(start + b, start + b + n, dtype=torch.int64, device=device)
        z = _splitmix64_torch(idx + key)
        sign = _lsr(z, 63) << 31
        e = torch.remainder(_lsr(z, 23), FULLMANT_BINADES)
        bits = sign | ((127 - e) << 23) | (z & 0x7FFFFF)
        # low 32 bits as a signed int32 (two's complement) -> the fp32 pattern
        ov[b:b + n] = (bits - ((bits >> 31) & 1) * (1 << 32)).to(torch.int32)
    return out
