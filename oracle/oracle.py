"""CPU ORACLE for the vertex-contribution EC path -- TEST INFRASTRUCTURE ONLY.

Python face of ``oracle/ft_oracle.c`` (a plain-C restatement of the reference
package ``fieldtopo``) plus numpy restatements of the curve assembly.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import this module, and only as the checker
or the timed CPU baseline.  The product package never imports it.

Parity pin: ``tests/test_oracle_golden.py`` checks every function here against
``tests/golden/*.npz``, produced by importing the reference itself
(``tests/golden/gen_golden.py``).

Reference anchors:
  quantize_with_range      fields.py:20-33
  gather_2d_*              contrib2d.py:161-294
  gather_3d_*              contrib3d.py:241-458
  split_blocks             _parallel.py:8-24
  counts_at_levels         descriptors.py:153-161
  descriptor_curve         descriptors.py:169-178
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_BUILD = _HERE / "_build"
_LIB_PATH = _BUILD / "libft_oracle.so"
_lib = None

DTYPE_CODES = {np.dtype(np.int32): 0, np.dtype(np.uint8): 1, np.dtype(np.uint16): 2,
               np.dtype(np.float32): 3, np.dtype(np.float64): 4}


def build(force=False):
    """Compile ft_oracle.c into oracle/_build/libft_oracle.so (gcc, -O2,
    -ffp-contract=off so float64 quantize rounds exactly like numpy)."""
    src = _HERE / "ft_oracle.c"
    if not force and _LIB_PATH.exists() and _LIB_PATH.stat().st_mtime >= src.stat().st_mtime:
        return _LIB_PATH
    _BUILD.mkdir(exist_ok=True)
    tmp = _LIB_PATH.with_suffix(f".{os.getpid()}.tmp")
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                           "-shared", "-pthread", "-o", str(tmp), str(src), "-lm"])
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB_PATH))
        i64, i32, dbl, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p
        L.ft_oracle_quantize.argtypes = [vp, ctypes.c_int, i64, dbl, dbl, i32, vp]
        L.ft_oracle_quantize.restype = None
        L.ft_oracle_gather2d.argtypes = [vp, ctypes.c_int, ctypes.c_int, dbl, dbl, i64, i64,
                                         i32, i64, i64, ctypes.c_int, vp, vp]
        L.ft_oracle_gather2d.restype = ctypes.c_int
        L.ft_oracle_gather3d.argtypes = [vp, ctypes.c_int, ctypes.c_int, dbl, dbl, i64, i64,
                                         i64, i32, i64, i64, ctypes.c_int, vp, vp]
        L.ft_oracle_gather3d.restype = ctypes.c_int
        L.ft_oracle_accum3d.argtypes = [vp, i32, vp, vp]
        L.ft_oracle_accum3d.restype = ctypes.c_int
        L.ft_oracle_split_blocks.argtypes = [i64, ctypes.c_int, vp, vp]
        L.ft_oracle_split_blocks.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def quantize_with_range(raw, lo, hi, max_level):
    """fields.py:20-33 restated in C (float64, round half up, clip)."""
    if max_level < 1:
        raise ValueError("max_level must be >= 1")
    a = np.ascontiguousarray(raw)
    if a.dtype not in DTYPE_CODES:
        a = a.astype(np.float64)
    out = np.empty(a.shape, np.int32)
    lib().ft_oracle_quantize(_ptr(a), DTYPE_CODES[a.dtype], a.size, float(lo), float(hi),
                             int(max_level), _ptr(out))
    return out


def quantize(raw, max_level):
    """fields.py:36-45: range from the data's own min and max."""
    a = np.asarray(raw)
    if a.size == 0:
        raise ValueError("empty field")
    return quantize_with_range(a, float(a.min()), float(a.max()), max_level)


def split_blocks(total, workers):
    lo = np.zeros(max(workers, 1), np.int64)
    hi = np.zeros(max(workers, 1), np.int64)
    nb = lib().ft_oracle_split_blocks(int(total), int(workers), _ptr(lo), _ptr(hi))
    if nb < 0:
        raise ValueError("workers must be >= 1")
    return [(int(a), int(b)) for a, b in zip(lo[:nb], hi[:nb])]


def _prep(x, value_range):
    a = np.ascontiguousarray(x)
    if a.dtype not in DTYPE_CODES:
        raise TypeError(f"unsupported dtype {a.dtype}")
    if value_range is None:
        if a.dtype not in (np.int32, np.uint8, np.uint16):
            raise TypeError("float input needs value_range=(lo, hi)")
        return a, 0, 0.0, 0.0
    return a, 1, float(value_range[0]), float(value_range[1])


def gather2d(x, max_level, value_range=None, workers=1, rows=None):
    """Reference 2D gather (contrib2d.py:161-294) -> (q_in, q_out) uint64 (5, M+2).

    ``x`` holds integer levels, or raw samples quantized on the fly with
    quantize_with_range(lo, hi, M) when ``value_range`` is given.  ``rows``
    restricts to vertex rows [a, b) (slab oracle)."""
    a, q, lo, hi = _prep(x, value_range)
    H, W = a.shape
    M = int(max_level)
    r0, r1 = rows if rows is not None else (0, H + 1)
    q_in = np.zeros((5, M + 2), np.uint64)
    q_out = np.zeros_like(q_in)
    rc = lib().ft_oracle_gather2d(_ptr(a), DTYPE_CODES[a.dtype], q, lo, hi, H, W, M, r0, r1,
                                  int(workers), _ptr(q_in), _ptr(q_out))
    if rc == 1:
        raise ValueError("workers must be >= 1")
    return q_in, q_out


def gather3d(x, max_level, value_range=None, workers=1, rows=None):
    """Reference 3D gather (contrib3d.py:241-458) -> (q_in, q_out) uint64 (21, M+2)."""
    a, q, lo, hi = _prep(x, value_range)
    H, W, D = a.shape
    M = int(max_level)
    r0, r1 = rows if rows is not None else (0, H + 1)
    q_in = np.zeros((21, M + 2), np.uint64)
    q_out = np.zeros_like(q_in)
    rc = lib().ft_oracle_gather3d(_ptr(a), DTYPE_CODES[a.dtype], q, lo, hi, H, W, D, M, r0, r1,
                                  int(workers), _ptr(q_in), _ptr(q_out))
    if rc == 1:
        raise ValueError("workers must be >= 1")
    if rc == 2:
        raise RuntimeError("3D neighborhood outside the configuration table")
    return q_in, q_out


def accum3d(vals, max_level):
    """One 3D vertex neighbourhood (contrib3d.py:220-238)."""
    v = np.ascontiguousarray(vals, np.int64)
    M = int(max_level)
    q_in = np.zeros((21, M + 2), np.uint64)
    q_out = np.zeros_like(q_in)
    if lib().ft_oracle_accum3d(_ptr(v), M, _ptr(q_in), _ptr(q_out)):
        raise RuntimeError("3D neighborhood outside the configuration table")
    return q_in, q_out


def counts_at_levels(q_in, q_out, max_level):
    """descriptors.py:153-161."""
    births = np.cumsum(q_in.astype(np.int64), axis=1)
    deaths = np.cumsum(q_out.astype(np.int64), axis=1)
    return (births - deaths)[:, : max_level + 1]


def descriptor_numerators(q_in, q_out, max_level, eighths):
    """descriptors.py:169-178: eighths @ counts (int64 numerators over 8)."""
    return np.asarray(eighths, np.int64) @ counts_at_levels(q_in, q_out, max_level)


# Built-in weight tables in eighths, type order as the reference
# (descriptors.py:83-97).  Pinned against the reference in the golden tests.
BUILTIN_2D = {
    ("ec", "8C"): (2, 0, -4, -2, 0),
    ("ec", "4C"): (2, 0, 4, -2, 0),
    ("perimeter", None): (8, 8, 16, 8, 0),
    ("area", None): (2, 4, 4, 6, 8),
}
BUILTIN_3D = {
    ("ec", "26C"): (1, 0, -2, -6, -1, -3, -1, 0, -2, -2, 0, 0, 4, -1, 1, 3, 0, 2, 2, 1, 0),
    ("perimeter", None): (12, 8, 24, 24, 12, 20, 36, 0, 24, 16, 24, 16, 48, 12, 20, 36, 8,
                          24, 24, 12, 0),
    ("surface-area", None): (6, 8, 12, 12, 10, 14, 18, 8, 12, 12, 16, 16, 24, 10, 14, 18, 8,
                             12, 12, 6, 0),
    ("volume", None): (1, 2, 2, 2, 3, 3, 3, 4, 4, 4, 4, 4, 4, 5, 5, 5, 6, 6, 6, 7, 8),
}
