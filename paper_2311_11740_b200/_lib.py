"""ctypes binding of the C ABI in ``include/fieldtopo_b200.h``.

The CUDA library is the only compute path of this package: if it is missing
or cannot be loaded, every entry point raises -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import threading

from . import build as _build
from ._tables import ClassificationError

FT_I32, FT_U8, FT_U16, FT_F32, FT_F64 = 0, 1, 2, 3, 4
FT_Q_IDENTITY, FT_Q_TABLE, FT_Q_TABLE_ROBUST, FT_Q_POW2 = 0, 1, 2, 3
FT_ERR_ARG, FT_ERR_CLASSIFY, FT_ERR_INTERNAL, FT_ERR_CUDA_BASE = 1, 2, 3, 1000

EXPORTS = ("ft_hist2d", "ft_hist3d", "ft_lattice2d", "ft_lattice3d", "ft_lines3d", "ft_lines3d_ok", "ft_lines2d", "ft_lines2d_ok", "ft_finalize", "ft_curves", "ft_class_weights", "ft_tables",
           "ft_quantize", "ft_quantize_probe", "ft_minmax", "ft_key_to_double", "ft_key64_to_double", "ft_version",
           "ft_stream_begin", "ft_stream_push", "ft_stream_end", "ft_multi_gather3d", "ft_bmp_decode",
           "ft_classify_status", "ft_debug_trap_tables")
FT_KIND_MAP, FT_KIND_FUSED = 0, 1


class ft_quant(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("negate", ctypes.c_int32), ("scale", ctypes.c_float),
                ("bias", ctypes.c_float), ("thresholds", ctypes.c_void_p),
                ("lo", ctypes.c_double), ("hi", ctypes.c_double)]


class ft_window(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("first", ctypes.c_int64),
                ("count", ctypes.c_int64), ("batch", ctypes.c_int64), ("batch_stride", ctypes.c_int64)]


class ft_slab(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("win", ft_window), ("v0", ctypes.c_int64), ("v1", ctypes.c_int64),
                ("quant", ft_quant), ("hist", ctypes.c_void_p)]


_lock = threading.Lock()
_lib = None


def load(build_if_missing=True):
    """Load (building first when stale and nvcc is available) the library."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = _build.LIB
        if build_if_missing and not _build.up_to_date():
            try:
                _build.build()
            except RuntimeError:
                if not path.exists():
                    raise
        if not path.exists():
            raise RuntimeError(f"fieldtopo-b200 CUDA library not built ({path}); "
                               "run `python -m paper_2311_11740_b200.build`")
        L = ctypes.CDLL(str(path))
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        P = ctypes.POINTER
        L.ft_hist2d.argtypes = [P(ft_window), i64, i64, i64, i64, P(ft_quant), i32, vp, vp]
        L.ft_hist3d.argtypes = [P(ft_window), i64, i64, i64, i64, i64, P(ft_quant), i32, vp, vp]
        L.ft_lattice3d.argtypes = [P(ft_window), i64, i64, i64, i64, i64, P(ft_quant), i32, vp, vp]
        L.ft_lattice2d.argtypes = [P(ft_window), i64, i64, i64, i64, P(ft_quant), i32, i32, vp, vp]
        L.ft_lines3d.argtypes = [P(ft_window), i64, i64, i64, i64, i64, P(ft_quant), i32, vp, vp]
        L.ft_lines3d_ok.argtypes = [i32]
        L.ft_lines2d.argtypes = [P(ft_window), i64, i64, i64, i64, P(ft_quant), i32, vp, vp]
        L.ft_lines2d_ok.argtypes = [i32]
        L.ft_finalize.argtypes = [i32, i32, i64, vp, vp, vp, i32, vp, vp, vp]
        L.ft_curves.argtypes = [vp, i32, i32, i64, i32, vp, vp, vp]
        L.ft_class_weights.argtypes = [i32, vp, vp]
        L.ft_tables.argtypes = [i32, vp, vp, vp]
        L.ft_quantize.argtypes = [vp, i32, i64, P(ft_quant), i32, vp, vp]
        L.ft_quantize_probe.argtypes = [vp, i32, i64, P(ft_quant), i32, i32, vp, vp]
        L.ft_minmax.argtypes = [vp, i32, i64, vp, vp]
        L.ft_key_to_double.argtypes = [i32, ctypes.c_uint32]
        L.ft_key_to_double.restype = ctypes.c_double
        L.ft_key64_to_double.argtypes = [ctypes.c_uint64]
        L.ft_key64_to_double.restype = ctypes.c_double
        L.ft_version.restype = ctypes.c_char_p
        L.ft_stream_begin.argtypes = [i32, i64, i64, i64, i32, P(ft_quant), i32, i32, i64, vp, vp, P(vp)]
        L.ft_stream_push.argtypes = [vp, vp, i64]
        L.ft_bmp_decode.argtypes = [vp, i64, i64, i64, i32, vp, vp]
        L.ft_classify_status.argtypes = [vp]
        L.ft_debug_trap_tables.argtypes = [i32]
        L.ft_stream_end.argtypes = [vp]
        L.ft_multi_gather3d.argtypes = [P(ft_slab), i32, i64, i64, i64, i32, i32, P(i32)]
        for name in EXPORTS:
            if name not in ("ft_key_to_double", "ft_key64_to_double", "ft_version"):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
        return L


def check(rc, what=""):
    """Map a C-ABI return code onto the reference's exception types."""
    if rc == 0:
        return
    if rc == FT_ERR_ARG:
        raise ValueError(f"{what}: invalid argument")
    if rc == FT_ERR_CLASSIFY:
        raise ClassificationError("3D neighborhood outside the configuration table")
    if rc == FT_ERR_INTERNAL:
        raise RuntimeError(f"{what}: unsupported device state (shared-memory layout)")
    if rc >= FT_ERR_CUDA_BASE:
        raise RuntimeError(f"{what}: CUDA error {rc - FT_ERR_CUDA_BASE}")
    raise RuntimeError(f"{what}: error code {rc}")
