"""Gather drivers: source -> device histogram (map or fused-curve kind).

Replaces the reference drivers gather_{2d,3d}_{serial,parallel} and their
sliding-window streaming loops (contrib2d.py:235-294, contrib3d.py:392-458,
_parallel.py:8-33) with:

* resident sources (``MemorySource``, ``DeviceSource``): one launch per vertex
  row block on the field already in HBM;
* streamed sources (``ArraySource``, ``BmpSource``, ``RawVolumeSource``):
  chunks of cell rows/planes in pinned host memory are copied to two device
  buffers on a side stream, so the H2D of chunk c+1 overlaps the kernel on
  chunk c.  Chunk c covers vertex rows [a, b) and holds cell rows
  [a-2, b-1]; the low halo rows are simply re-sent.  A source that is
  already a pinned torch tensor is copied straight from its own pages; any
  other source is read into two pinned staging buffers first;
* several GPUs in one process (``devices=[...]``): vertex-row slabs per GPU
  like split_blocks, histograms summed after the join.

``kind`` selects the kernel family: "map" = transition-class histograms
(ft_hist2d/3d -> contribution maps), "lattice" = element histograms
(ft_lattice2d/3d -> curves only), "lines" = the 3D line-decomposition rows
(ft_lines3d -> EC / surface-area / volume curves only).  Every path gives the same histogram bit
for bit: integer sums commute.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import engine
from ._parallel import LOW_HALO, held_rows, split_blocks

DEFAULT_CHUNK_BYTES = 256 << 20


@dataclass(frozen=True)
class Kind:
    name: str = "map"
    maxes: bool = False

    def new(self, ndim, M, device, batch=1):
        if self.name == "map":
            return engine.new_hist(ndim, M, device, batch)
        if self.name == "lines":
            return engine.new_lines_hist(M, device)
        return engine.new_lattice_hist(ndim, M, device, batch)

    def launch(self, ndim, x, shape, M, quant, rows, first=0, hist=None, batch=1, batch_stride=0):
        if self.name == "map":
            return engine.launch_hist(ndim, x, shape, M, quant, rows=rows, first=first, hist=hist, batch=batch,
                                      batch_stride=batch_stride)
        if self.name == "lines":
            return engine.launch_lines(x, shape, M, quant, rows=rows, first=first, hist=hist)
        return engine.launch_lattice(ndim, x, shape, M, quant, rows=rows, first=first, hist=hist, batch=batch,
                                     batch_stride=batch_stride, maxes=self.maxes)


MAP = Kind("map")


def _torch_dtype(np_dtype):
    t = engine.torch()
    return {np.dtype(np.int32): t.int32, np.dtype(np.uint8): t.uint8, np.dtype(np.uint16): t.uint16,
            np.dtype(np.float32): t.float32}[np.dtype(np_dtype)]


def resident_hist(src, ndim, device, rows, workers=1, hist=None, kind=MAP):
    x, quant = src.device_field(device)
    if x.device != device:
        raise ValueError(f"the source's field lives on {x.device}, not on {device}")
    if hist is None:
        hist = kind.new(ndim, src.max_level, device)
    v0, v1 = rows
    for a, b in split_blocks(v1 - v0, workers):
        kind.launch(ndim, x, src.shape, src.max_level, quant, (v0 + a, v0 + b), hist=hist)
    return hist


def stream_hist(src, ndim, device, rows, chunk_bytes=DEFAULT_CHUNK_BYTES, hist=None, kind=MAP):
    """Double-buffered pinned-host -> HBM streaming of a source's rows/planes."""
    with engine.on_device(device):  # streams and events belong to ``device``
        return _stream_hist(src, ndim, device, rows, chunk_bytes, hist, kind)


def _stream_hist(src, ndim, device, rows, chunk_bytes, hist, kind):
    t = engine.torch()
    H = src.height
    M = src.max_level
    row_elems = src.width * (src.depth if ndim == 3 else 1)
    itemsize = np.dtype(src.dtype).itemsize
    tdt = _torch_dtype(src.dtype)
    cap = max(LOW_HALO + 1, int(chunk_bytes // max(1, row_elems * itemsize)))  # cell rows per buffer
    cap = min(cap, H + 1)
    vpc = max(1, cap - LOW_HALO)  # vertex rows per chunk (LOW_HALO halo rows re-sent)
    if hist is None:
        hist = kind.new(ndim, M, device)
    host = getattr(src, "pinned_rows", None)  # a pinned torch tensor (rows, ...) or None
    if host is None:
        staging = [t.empty(cap * row_elems, dtype=tdt, pin_memory=True) for _ in range(2)]
        src.note_resident(2 * cap * row_elems * itemsize)
    dbuf = [t.empty(cap * row_elems, dtype=tdt, device=device) for _ in range(2)]
    compute = t.cuda.current_stream(device)
    copy = t.cuda.Stream(device)
    copied = [t.cuda.Event() for _ in range(2)]
    done = [None, None]
    v0, v1 = rows
    for c, a in enumerate(range(v0, v1, vpc)):
        b = min(a + vpc, v1)
        s = c & 1
        r0, r1 = held_rows(a, b, H)
        n = (r1 - r0) * row_elems
        if host is None:
            if done[s] is not None:
                done[s].synchronize()  # staging[s] free again
            src.read_rows(r0, r1, staging[s].numpy()[:n])
            chunk = staging[s][:n]
        else:
            chunk = host[r0 - src.pinned_first:r1 - src.pinned_first].reshape(-1)
        with t.cuda.stream(copy):
            if done[s] is not None:
                copy.wait_event(done[s])  # dbuf[s] consumed by the previous kernel
            dbuf[s][:n].copy_(chunk, non_blocking=True)
            copied[s].record(copy)
        compute.wait_event(copied[s])
        view = dbuf[s][:n].view((r1 - r0,) + tuple(src.shape[1:]))
        kind.launch(ndim, view, src.shape, M, src.quant, (a, b), first=r0, hist=hist)
        ev = t.cuda.Event()
        ev.record(compute)
        done[s] = ev
    return hist


def source_hist(src, ndim, device=None, workers=1, rows=None, chunk_bytes=DEFAULT_CHUNK_BYTES, kind=MAP):
    """Histogram of ``src`` for vertex rows ``rows`` on one GPU."""
    if device is None and src.mode == "device":
        dev = src.tensor.device  # a resident field is processed where it lives
    else:
        dev = engine.default_device(device)
    rows = rows if rows is not None else (0, src.height + 1)
    if src.mode in ("in-memory", "device"):
        return resident_hist(src, ndim, dev, rows, workers, kind=kind)
    return stream_hist(src, ndim, dev, rows, chunk_bytes, kind=kind)


def multi_device_hist(src, ndim, devices, chunk_bytes=DEFAULT_CHUNK_BYTES, kind=MAP):
    """Vertex-row slabs over several GPUs of this process; returns the summed
    histogram on devices[0].  Resident host fields upload only each slab's
    planes plus the one-plane halo."""
    devs = [engine.default_device(d) for d in devices]
    blocks = split_blocks(src.height + 1, len(devs))
    parts = []
    for dev, (a, b) in zip(devs, blocks):
        if src.mode == "in-memory":
            r0, r1 = held_rows(a, b, src.height)
            x = engine.to_device(src.field.values[r0:r1], dev)
            h = kind.new(ndim, src.max_level, dev)
            parts.append(kind.launch(ndim, x, src.shape, src.max_level, engine.QuantSpec.identity(), (a, b),
                                     first=r0, hist=h))
        elif src.mode == "device":
            raise ValueError("a DeviceSource lives on one GPU; use devices=None")
        else:
            parts.append(stream_hist(src, ndim, dev, (a, b), chunk_bytes, kind=kind))
    total = parts[0]
    for p in parts[1:]:
        total += p.to(devs[0])
    return total
