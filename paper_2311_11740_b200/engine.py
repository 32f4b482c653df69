"""Device driver: field residency, kernel launches, finalize.

PyTorch supplies device memory, streams and ``torch.distributed`` plumbing;
every byte of the hot path is computed by the CUDA library through the C ABI
(``_lib``).  Histograms are int64 tensors on the device that the library
treats as uint64 (counts never exceed 2**63).
"""

from __future__ import annotations

import ctypes
import warnings
import numpy as np

from . import _lib
from ._tables import TRANSITIONS_2D, TRANSITIONS_3D
from .quant import QuantSpec, device_struct

NCLASS = {2: 6, 3: 40}
NTYPE = {2: 5, 3: 21}

_TORCH_DTYPE_CODES = None


def torch():
    import torch as _t
    return _t


def _codes():
    global _TORCH_DTYPE_CODES
    if _TORCH_DTYPE_CODES is None:
        t = torch()
        _TORCH_DTYPE_CODES = {t.int32: _lib.FT_I32, t.uint8: _lib.FT_U8, t.uint16: _lib.FT_U16,
                              t.float32: _lib.FT_F32, t.float64: _lib.FT_F64}
    return _TORCH_DTYPE_CODES


def dtype_code(tensor):
    try:
        return _codes()[tensor.dtype]
    except KeyError:
        raise TypeError(f"unsupported field dtype {tensor.dtype}; use int32 levels, uint8, "
                        "uint16 or float32") from None


def default_device(device=None):
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("fieldtopo-b200 needs a CUDA device (B200, sm_100a); none is visible")
    if device is None:
        return t.device("cuda", t.cuda.current_device())
    d = t.device(device)
    if d.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {d}")
    return d if d.index is not None else t.device("cuda", t.cuda.current_device())


def _stream_ptr(device):
    return ctypes.c_void_p(torch().cuda.current_stream(device).cuda_stream)


def on_device(device):
    """Make ``device`` the thread's current CUDA device for a library call.

    The C library takes the device from the calling thread (rank tables, SM
    count, kernel attributes, the launch itself) and the stream handle of
    torch's default stream is NULL, so every call that touches a tensor on
    cuda:N must run with cuda:N current (cuda:1 tensors launched
    from a cuda:0 thread would fault or race)."""
    return torch().cuda.device(device)


def _rows_held(ndim, x, batch):
    """Rows (2D) / planes (3D) the window tensor holds: an (N, H, W) image
    stack holds H rows for any N, including N == 1."""
    return x.shape[-2] if ndim == 2 and x.dim() == 3 else x.shape[0]


def to_device(array, device, pinned=True):
    """numpy/torch array -> contiguous CUDA tensor (pinned-staged H2D)."""
    t = torch()
    if isinstance(array, t.Tensor):
        x = array
    else:
        a = np.ascontiguousarray(array)
        if a.dtype == np.int64:
            a = a.astype(np.int32)
        with warnings.catch_warnings():  # read-only Field arrays: only ever read
            warnings.simplefilter("ignore", UserWarning)
            x = t.from_numpy(a)
        if pinned and x.numel() * x.element_size() >= (1 << 20):
            x = x.pin_memory()
    return x.to(device, non_blocking=True).contiguous()


def new_hist(ndim, M, device, batch=1):
    shape = (NCLASS[ndim], M + 2) if batch == 1 else (batch, NCLASS[ndim], M + 2)
    return torch().zeros(shape, dtype=torch().int64, device=device)


def launch_hist(ndim, x, shape, M, quant, rows=None, first=0, hist=None, batch=1, batch_stride=0):
    """Accumulate transition histograms of vertex rows ``rows`` = [v0, v1).

    ``x``: CUDA tensor holding rows/planes [first, first + count) of a field of
    global shape ``shape`` ((H, W) or (H, W, D)); for ``batch`` > 1 (2D) the
    images are ``batch_stride`` elements apart."""
    L = _lib.load()
    dev = x.device
    H = shape[0]
    v0, v1 = rows if rows is not None else (0, H + 1)
    if hist is None:
        hist = new_hist(ndim, M, dev, batch)
    count = _rows_held(ndim, x, batch)
    win = _lib.ft_window(ctypes.c_void_p(x.data_ptr()), dtype_code(x), int(first), int(count),
                         int(batch), int(batch_stride))
    with on_device(dev):
        qs, keep = device_struct(quant, dev)
        rc = _hist_call(L, ndim, win, H, shape, v0, v1, qs, M, hist, _stream_ptr(dev))
    del keep
    _lib.check(rc, f"ft_hist{ndim}d")
    return hist


def _hist_call(L, ndim, win, H, shape, v0, v1, qs, M, hist, st):
    if ndim == 2:
        return L.ft_hist2d(ctypes.byref(win), H, shape[1], v0, v1, ctypes.byref(qs), M,
                           ctypes.c_void_p(hist.data_ptr()), st)
    return L.ft_hist3d(ctypes.byref(win), H, shape[1], shape[2], v0, v1, ctypes.byref(qs), M,
                       ctypes.c_void_p(hist.data_ptr()), st)


def new_lattice_hist(ndim, M, device, batch=1):
    shape = (4, M + 2) if batch == 1 else (batch, 4, M + 2)
    return torch().zeros(shape, dtype=torch().int64, device=device)


def _use_lines2d(kernel, batch):
    """ft_lines2d or ft_lattice2d for 2D rows 0..2.  ft_lines2d is the default:
    measured on B200 (ncu kernel durations, profiles/r01/lines2d_notes.md) it
    beats the lattice kernel on one large image (C2: 85 vs 90 us) and on
    batches (C3: 715 vs 779 us).  ``kernel`` "lines" / "lattice" forces one."""
    return kernel != "lattice"


def launch_lattice(ndim, x, shape, M, quant, rows=None, first=0, hist=None, batch=1, batch_stride=0,
                   maxes=False, kernel="auto"):
    """Accumulate the fused-curve element histograms (ft_lattice2d/3d) of
    lattice rows ``rows`` = [v0, v1); arguments as ``launch_hist``.  2D
    without vertex maxes may go to ft_lines2d (same rows, _use_lines2d)."""
    L = _lib.load()
    dev = x.device
    H = shape[0]
    v0, v1 = rows if rows is not None else (0, H + 1)
    if hist is None:
        hist = new_lattice_hist(ndim, M, dev, batch)
    count = _rows_held(ndim, x, batch)
    win = _lib.ft_window(ctypes.c_void_p(x.data_ptr()), dtype_code(x), int(first), int(count),
                         int(batch), int(batch_stride))
    with on_device(dev):
        qs, keep = device_struct(quant, dev)
        st = _stream_ptr(dev)
        if ndim == 2 and not maxes and lines2d_ok(M) and _use_lines2d(kernel, batch):
            # rows 0..2 by line decomposition (ft_lines2d): fewer shared atomics
            name = "ft_lines2d"
            rc = L.ft_lines2d(ctypes.byref(win), H, shape[1], v0, v1, ctypes.byref(qs), M,
                              ctypes.c_void_p(hist.data_ptr()), st)
        elif ndim == 2:
            name = "ft_lattice2d"
            rc = L.ft_lattice2d(ctypes.byref(win), H, shape[1], v0, v1, ctypes.byref(qs), M, int(maxes),
                                ctypes.c_void_p(hist.data_ptr()), st)
        else:
            name = "ft_lattice3d"
            rc = L.ft_lattice3d(ctypes.byref(win), H, shape[1], shape[2], v0, v1, ctypes.byref(qs), M,
                                ctypes.c_void_p(hist.data_ptr()), st)
    del keep
    _lib.check(rc, name)
    return hist


def new_lines_hist(M, device):
    return torch().zeros((3, M + 2), dtype=torch().int64, device=device)


def launch_lines(x, shape, M, quant, rows=None, first=0, hist=None):
    """Accumulate the 3D line-decomposition rows (C, F, V - E; ft_lines3d) of
    lattice rows ``rows`` = [v0, v1); arguments as ``launch_hist``."""
    L = _lib.load()
    dev = x.device
    H = shape[0]
    v0, v1 = rows if rows is not None else (0, H + 1)
    if hist is None:
        hist = new_lines_hist(M, dev)
    win = _lib.ft_window(ctypes.c_void_p(x.data_ptr()), dtype_code(x), int(first), int(x.shape[0]), 1, 0)
    with on_device(dev):
        qs, keep = device_struct(quant, dev)
        rc = L.ft_lines3d(ctypes.byref(win), H, shape[1], shape[2], v0, v1, ctypes.byref(qs), M,
                          ctypes.c_void_p(hist.data_ptr()), _stream_ptr(dev))
    del keep
    _lib.check(rc, "ft_lines3d")
    return hist


def lines2d_ok(M):
    """Whether ft_lines2d takes this level count."""
    return bool(_lib.load().ft_lines2d_ok(int(M)))


def lines_ok(M):
    """Whether ft_lines3d takes this level count (16-bit packed row offsets)."""
    return bool(_lib.load().ft_lines3d_ok(int(M)))


def lattice_ok(ndim, shape, M, x=None):
    """Whether the fused lattice kernels accept this field (levels * 4 must
    fit the 16-bit packed lanes)."""
    return (M + 1) * 4 <= 0xFFFF


_row_w_cache = {}


def _row_weights(row_w, dev):
    """Row weights on ``dev``, uploaded once per (table, device): a pageable
    H2D copy per call would block the host until the stream drains and leave
    the GPU idle between back-to-back launches."""
    a = np.ascontiguousarray(np.asarray(row_w, np.int64))
    key = (a.shape, a.tobytes(), str(dev))
    w = _row_w_cache.get(key)
    if w is None:
        w = torch().from_numpy(a.copy()).to(dev)
        _row_w_cache[key] = w
    return w


def curves_from_rows(hist, M, row_w):
    """Device weighted prefix scan of histogram rows -> int64 numerators
    [n_desc, M+1] (or [batch, n_desc, M+1])."""
    t = torch()
    L = _lib.load()
    dev = hist.device
    batch = hist.shape[0] if hist.dim() == 3 else 1
    n_rows = hist.shape[-2]
    w = _row_weights(row_w, dev)
    n_desc = w.shape[0]
    # a batched (3D) histogram keeps its batch axis, also for one image
    out = t.empty((n_desc, M + 1) if hist.dim() == 2 else (batch, n_desc, M + 1), dtype=t.int64, device=dev)
    with on_device(dev):
        rc = L.ft_curves(ctypes.c_void_p(hist.data_ptr()), n_rows, M, batch, n_desc,
                         ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(out.data_ptr()), _stream_ptr(dev))
    _lib.check(rc, "ft_curves")
    return out


def class_weights(ndim, eighths):
    tables = TRANSITIONS_3D if ndim == 3 else TRANSITIONS_2D
    w = np.asarray(eighths, np.int64)
    if w.shape != (tables.n_types,):
        raise ValueError(f"{ndim}D table needs {tables.n_types} weights")
    out = np.zeros(tables.n_classes, np.int64)
    _lib.check(_lib.load().ft_class_weights(ndim, w.ctypes.data, out.ctypes.data), "ft_class_weights")
    return out


def finalize(ndim, M, hist, maps=True, tables=()):
    """Device q_in/q_out (uint64 as int64, or None) and numerators [n_desc, M+1]."""
    t = torch()
    L = _lib.load()
    dev = hist.device
    batch = hist.shape[0] if hist.dim() == 3 else 1
    T = NTYPE[ndim]
    shp = (T, M + 2) if hist.dim() == 2 else (batch, T, M + 2)
    q_in = t.empty(shp, dtype=t.int64, device=dev) if maps else None
    q_out = t.empty(shp, dtype=t.int64, device=dev) if maps else None
    n_desc = len(tables)
    cw = num = None
    if n_desc:
        cw = t.from_numpy(np.stack([class_weights(ndim, w) for w in tables])).to(dev)
        num = t.empty((n_desc, M + 1) if hist.dim() == 2 else (batch, n_desc, M + 1), dtype=t.int64, device=dev)
    ptr = lambda a: ctypes.c_void_p(a.data_ptr()) if a is not None else None  # noqa: E731
    with on_device(dev):
        rc = L.ft_finalize(ndim, M, batch, ptr(hist), ptr(q_in), ptr(q_out), n_desc, ptr(cw), ptr(num),
                           _stream_ptr(dev))
    _lib.check(rc, "ft_finalize")
    return q_in, q_out, num


def check_classification(device):
    """Raise ClassificationError if a 3D map kernel on ``device`` met a
    neighbourhood outside the configuration table since the last check
    (ft_classify_status; waits for the device's current stream)."""
    with on_device(device):
        _lib.check(_lib.load().ft_classify_status(_stream_ptr(device)), "ft_hist3d")


def curves_from_maps(q_in, q_out, M, eighths_list, device):
    """descriptor_curve / counts_at_levels on device: weighted prefix scan of
    the rows (q_in; q_out) with weights (w; -w)."""
    t = torch()
    L = _lib.load()
    rows = np.concatenate([np.asarray(q_in, np.uint64), np.asarray(q_out, np.uint64)]).view(np.int64)
    w = np.asarray(eighths_list, np.int64)
    row_w = np.concatenate([w, -w], axis=1)
    r = t.from_numpy(np.ascontiguousarray(rows)).to(device)
    rw = t.from_numpy(np.ascontiguousarray(row_w)).to(device)
    out = t.empty((len(w), M + 1), dtype=t.int64, device=device)
    with on_device(device):
        rc = L.ft_curves(ctypes.c_void_p(r.data_ptr()), rows.shape[0], M, 1, len(w),
                         ctypes.c_void_p(rw.data_ptr()), ctypes.c_void_p(out.data_ptr()), _stream_ptr(device))
    _lib.check(rc, "ft_curves")
    return out.cpu().numpy()


def quantize_device(x, quant, M):
    """Standalone device quantize -> int32 tensor."""
    t = torch()
    L = _lib.load()
    out = t.empty(x.shape, dtype=t.int32, device=x.device)
    with on_device(x.device):
        qs, keep = device_struct(quant, x.device, f64=x.dtype == t.float64)
        rc = L.ft_quantize(ctypes.c_void_p(x.data_ptr()), dtype_code(x), x.numel(), ctypes.byref(qs), M,
                           ctypes.c_void_p(out.data_ptr()), _stream_ptr(x.device))
    del keep
    _lib.check(rc, "ft_quantize")
    return out


def minmax_device(x):
    """(min, max) of a CUDA tensor as Python floats (device reduction)."""
    t = torch()
    L = _lib.load()
    out = t.empty(4, dtype=t.int32, device=x.device)
    code = dtype_code(x)
    with on_device(x.device):
        rc = L.ft_minmax(ctypes.c_void_p(x.data_ptr()), code, x.numel(), ctypes.c_void_p(out.data_ptr()),
                         _stream_ptr(x.device))
    _lib.check(rc, "ft_minmax")
    raw = out.cpu().numpy()
    if code == _lib.FT_F64:
        k = raw.view(np.uint64)
        return L.ft_key64_to_double(int(k[0])), L.ft_key64_to_double(int(k[1]))
    k = raw.view(np.uint32)
    return L.ft_key_to_double(code, int(k[0])), L.ft_key_to_double(code, int(k[1]))


def as_uint64(t):
    """Device int64 histogram/map tensor -> host numpy uint64."""
    return t.cpu().numpy().view(np.uint64)


__all__ = ["launch_hist", "finalize", "curves_from_maps", "quantize_device", "minmax_device", "to_device",
           "default_device", "new_hist", "as_uint64", "class_weights", "QuantSpec"]


def stream_native(rows, shape, M, quant, kind="map", chunk_rows=64, push_rows=None, device=None, hist=None):
    """Histogram of a field pushed row block by row block through the native
    streaming engine (ft_stream_begin / push / end: the C-ABI twin of
    gather.stream_hist for non-Python callers).  ``rows``: the whole field
    as a host numpy array (pageable), a pinned / CPU torch tensor or a CUDA
    tensor -- it is only READ, ``push_rows`` rows per ft_stream_push."""
    t = torch()
    L = _lib.load()
    dev = default_device(device)
    ndim = len(shape)
    H, W = shape[0], shape[1]
    D = shape[2] if ndim == 3 else 1
    k = _lib.FT_KIND_MAP if kind == "map" else _lib.FT_KIND_FUSED
    if hist is None:
        hist = new_hist(ndim, M, dev) if kind == "map" else (new_lines_hist(M, dev) if ndim == 3
                                                            else new_lattice_hist(2, M, dev))
    if isinstance(rows, np.ndarray):
        a = np.ascontiguousarray(rows)
        ptr, code, row_bytes = a.ctypes.data, dtype_code(t.from_numpy(a[:1].copy())), a[0].nbytes
    else:
        a = rows.contiguous()
        ptr, code, row_bytes = a.data_ptr(), dtype_code(a), a[0].numel() * a.element_size()
    push_rows = push_rows or chunk_rows
    with on_device(dev):
        qs, keep = device_struct(quant, dev)
        h = ctypes.c_void_p()
        _lib.check(L.ft_stream_begin(ndim, H, W, D, code, ctypes.byref(qs), M, k, chunk_rows,
                                     ctypes.c_void_p(hist.data_ptr()), _stream_ptr(dev), ctypes.byref(h)),
                   "ft_stream_begin")
        try:
            for r in range(0, H, push_rows):
                n = min(push_rows, H - r)
                _lib.check(L.ft_stream_push(h, ctypes.c_void_p(ptr + r * row_bytes), n), "ft_stream_push")
        finally:
            rc = L.ft_stream_end(h)
        _lib.check(rc, "ft_stream_end")
    del keep, a
    return hist


def multi_gather_native(parts, shape, M, quant, kind="map"):
    """ft_multi_gather3d over ``parts`` = [(CUDA tensor of planes [r0, r1),
    r0, (v0, v1))] (one per slab, any devices); returns (per-slab histogram
    tensors, each holding the whole-field sum, used_nccl)."""
    L = _lib.load()
    H, W, D = shape
    k = _lib.FT_KIND_MAP if kind == "map" else _lib.FT_KIND_FUSED
    slabs = (_lib.ft_slab * len(parts))()
    keep, hists = [], []
    for s, (x, r0, (v0, v1)) in zip(slabs, parts):
        with on_device(x.device):
            qs, kt = device_struct(quant, x.device)
            h = new_hist(3, M, x.device) if kind == "map" else new_lines_hist(M, x.device)
        keep += [kt, x]
        hists.append(h)
        s.device = x.device.index
        s.win = _lib.ft_window(ctypes.c_void_p(x.data_ptr()), dtype_code(x), int(r0), int(x.shape[0]), 1, 0)
        s.v0, s.v1 = int(v0), int(v1)
        s.quant = qs
        s.hist = ctypes.c_void_p(h.data_ptr())
    torch().cuda.synchronize()  # histograms zeroed before the library's own streams use them
    used = ctypes.c_int32(0)
    _lib.check(L.ft_multi_gather3d(slabs, len(parts), H, W, D, M, k, ctypes.byref(used)), "ft_multi_gather3d")
    del keep
    return hists, bool(used.value)
