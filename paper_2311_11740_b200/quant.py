"""Exact device quantization: float32 threshold tables for quantize_with_range.

The reference maps samples onto levels with float64
``clip(floor((x - lo) * M / (hi - lo) + 0.5), 0, M)`` (fields.py:20-33).  The
map is monotone in x, so for float32-representable inputs (float32, uint8,
uint16) it is decided exactly by M thresholds: t_l = the smallest float32
whose reference level is >= l.  The kernels estimate the level with one
float32 FMA and fix it with one comparison on each side against the table
(``ft_common.cuh::to_level``).  The table itself is found here by bisection
over the ordered float32 space using the reference formula -- host work of
O(M * 32) evaluations, cached per (lo, hi, M, device).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _lib


def reference_levels(x, lo, hi, max_level):
    """The reference float64 formula (fields.py:29-33), used only to build
    threshold tables."""
    arr = np.asarray(x, dtype=np.float64)
    if hi == lo:
        return np.zeros(arr.shape, np.int64)
    scaled = (arr - lo) * float(max_level) / (hi - lo)
    return np.clip(np.floor(scaled + 0.5), 0, max_level).astype(np.int64)


def _f32_from_key(k):
    k = np.asarray(k, np.int64)
    u = np.where(k >= 0x80000000, k - 0x80000000, ~k & 0xFFFFFFFF).astype(np.uint32)
    return u.view(np.float32)


def _key_from_f32(f):
    u = np.asarray(f, np.float32).view(np.uint32).astype(np.int64)
    return np.where(u & 0x80000000, ~u & 0xFFFFFFFF, u | 0x80000000)


def _f64_from_key(k):
    k = np.asarray(k, np.int64)
    bits = np.where(k >= 0, k, (-(k + 1)) | np.int64(-0x8000000000000000))
    return bits.view(np.float64)


def _key_from_f64(f):
    b = np.asarray(f, np.float64).view(np.int64)
    return np.where(b >= 0, b, -(b & np.int64(0x7FFFFFFFFFFFFFFF)) - 1)


@lru_cache(maxsize=64)
def threshold_table_f64(lo, hi, max_level, negate=False):
    """Like threshold_table for float64 inputs: smallest double per level."""
    M = int(max_level)
    lo, hi = float(lo), float(hi)
    if negate:
        lo, hi = -lo, -hi
    t = np.full(M + 2, np.nan, np.float64)
    t[0] = -np.inf
    if hi == lo or M < 1:
        return t
    lvl = np.arange(1, M + 1, dtype=np.int64)
    a = np.full(M, int(_key_from_f64(-np.inf)), np.int64)
    b = np.full(M, int(_key_from_f64(np.inf)), np.int64)
    for _ in range(70):
        if np.all(a >= b):
            break
        mid = (a >> 1) + (b >> 1) + (a & b & 1)  # floor((a+b)/2), no int64 overflow
        ok = reference_levels(_f64_from_key(mid), lo, hi, M) >= lvl
        b = np.where(ok, mid, b)
        a = np.where(ok, a, mid + 1)
    t[1:M + 1] = _f64_from_key(b)
    return t


@lru_cache(maxsize=64)
def threshold_table(lo, hi, max_level, negate=False):
    """[-inf, t_1, ..., t_M, NaN] as float32 (length M + 2).

    With ``negate`` the table is over x' = -x for the equivalent increasing
    range (-lo, -hi); see DESIGN.md §5 for why that is exact."""
    M = int(max_level)
    lo, hi = float(lo), float(hi)
    if negate:
        lo, hi = -lo, -hi
    t = np.full(M + 2, np.nan, np.float32)
    t[0] = -np.inf
    if hi == lo or M < 1:
        return t
    lvl = np.arange(1, M + 1, dtype=np.int64)
    a = np.full(M, int(_key_from_f32(np.float32(-np.inf))), np.int64)
    b = np.full(M, int(_key_from_f32(np.float32(np.inf))), np.int64)
    # invariant: level(from_key(b)) >= l (true at +inf when hi > lo)
    for _ in range(40):
        if np.all(a >= b):
            break
        mid = (a + b) // 2
        ok = reference_levels(_f32_from_key(mid), lo, hi, M) >= lvl
        b = np.where(ok, mid, b)
        a = np.where(ok, a, mid + 1)
    t[1:M + 1] = _f32_from_key(b)
    return t


@dataclass(frozen=True)
class QuantSpec:
    """Level decoding of a raw buffer (mirrors the C struct ft_quant)."""

    mode: int
    negate: int = 0
    scale: float = 0.0
    bias: float = 0.0
    lo: float = 0.0
    hi: float = 0.0
    max_level: int = 0

    @staticmethod
    def identity():
        return QuantSpec(_lib.FT_Q_IDENTITY)

    @staticmethod
    def for_range(lo, hi, max_level):
        """quantize_with_range(x, lo, hi, max_level) for float32/u8/u16 x."""
        if max_level < 1:
            raise ValueError("max_level must be >= 1")
        lo, hi = float(lo), float(hi)
        if not (math.isfinite(lo) and math.isfinite(hi)):
            raise ValueError("quantization range must be finite")
        negate = hi < lo
        l2, h2 = (-lo, -hi) if negate else (lo, hi)
        if h2 == l2:
            return QuantSpec(_lib.FT_Q_TABLE, int(negate), 0.0, 0.0, lo, hi, int(max_level))
        scale = np.float32(max_level / (h2 - l2))
        # estimate floor(x*scale + bias) = floor(y - 0.5) lands on L or L-1
        bias = np.float32(-l2 * float(scale))
        # error of fmaf(x, scale, bias) against the float64 formula for x in
        # the window where the level is not clamped; beyond +-1 level the
        # kernel walks the table instead of a single correction step
        xmax = max(abs(l2), abs(h2)) + (h2 - l2)
        err = (xmax * abs(float(scale)) + abs(float(bias))) * 2.0 ** -22 + \
            abs(float(scale) * (h2 - l2) - max_level) + 1e-6
        mode = _lib.FT_Q_TABLE if err < 0.45 and not negate else _lib.FT_Q_TABLE_ROBUST
        if not negate and l2 == 0.0 and h2 > 0 and math.frexp(h2)[0] == 0.5 and max_level < (1 << 22):
            # lo = 0, hi = 2^p: scale = M / hi is exact and the reference's
            # float64 formula is exact for float32 inputs -> table-free mode
            # (the table still ships for kernels that use it)
            mode = _lib.FT_Q_POW2
            scale, bias = np.float32(max_level / h2), np.float32(0.0)
        return QuantSpec(mode, int(negate), float(scale), float(bias), lo, hi, int(max_level))

    @property
    def is_identity(self):
        return self.mode == _lib.FT_Q_IDENTITY

    def table(self, f64=False):
        fn = threshold_table_f64 if f64 else threshold_table
        return fn(self.lo, self.hi, self.max_level, bool(self.negate))


_dev_tables = {}


def device_struct(spec, device, f64=False):
    """(ft_quant ctypes struct, keep-alive tensor) for a launch on ``device``."""
    import torch

    if spec.is_identity:
        return _lib.ft_quant(_lib.FT_Q_IDENTITY, 0, 0.0, 0.0, None), None
    key = (spec.lo, spec.hi, spec.max_level, spec.negate, str(device), f64)
    t = _dev_tables.get(key)
    if t is None:
        t = torch.from_numpy(spec.table(f64)).to(device)
        _dev_tables[key] = t
    return _lib.ft_quant(spec.mode, spec.negate, spec.scale, spec.bias, ctypes.c_void_p(t.data_ptr()),
                         float(spec.lo), float(spec.hi)), t
