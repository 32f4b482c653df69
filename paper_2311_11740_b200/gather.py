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
  [a-2, b-1]; the two low halo rows are carried over from the previous
  chunk's buffer device-to-device, so every row crosses PCIe once
  (DESIGN.md §6).  A source that hands out pinned host rows (a pinned torch
  tensor, a pinned ring) is copied straight from its pages; any other source
  is read into two pinned staging buffers by a pool of host threads;
* several GPUs in one process (``devices=[...]``): vertex-row slabs per GPU
  like split_blocks, histograms summed after the join.

``kind`` selects the kernel family: "map" = transition-class histograms
(ft_hist2d/3d -> contribution maps), "lattice" = element histograms
(ft_lattice2d/3d -> curves only), "lines" = the 3D line-decomposition rows
(ft_lines3d -> EC / surface-area / volume curves only).  Every path gives the same histogram bit
for bit: integer sums commute.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
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


def _staging_threads():
    return max(1, min(16, os.cpu_count() or 1))


def _read_parallel(src, r0, r1, out, row_elems, pool):
    """src.read_rows over [r0, r1) into ``out`` (numpy view of a pinned
    buffer), split into row blocks read by the pool's threads: numpy copies
    and file preads release the GIL, so a multi-core host fills the pinned
    staging buffer at memory (or page-cache) speed instead of one core's."""
    n = r1 - r0
    parts = min(n, pool._max_workers)
    if parts <= 1 or not getattr(src, "parallel_reads", False):
        src.read_rows(r0, r1, out[: n * row_elems])
        return
    blocks = split_blocks(n, parts)
    futs = [pool.submit(src.read_rows, r0 + lo, r0 + hi, out[lo * row_elems:hi * row_elems]) for lo, hi in blocks]
    for f in futs:
        f.result()


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
    # a source that can hand out its rows as pinned host memory is copied
    # straight from those pages (a pinned torch tensor, a pinned ring of
    # planes); any other source is read into two pinned staging buffers
    window = getattr(src, "pinned_window", None)
    pool = None
    if window is None:
        staging = [t.empty(cap * row_elems, dtype=tdt, pin_memory=True) for _ in range(2)]
        src.note_resident(2 * cap * row_elems * itemsize)
        pool = cf.ThreadPoolExecutor(_staging_threads())
    dbuf = [t.empty(cap * row_elems, dtype=tdt, device=device) for _ in range(2)]
    compute = t.cuda.current_stream(device)
    copy = t.cuda.Stream(device)
    copied = [None, None]
    done = [None, None]
    v0, v1 = rows
    prev = None  # (buffer, r0, r1) of the previous chunk
    try:
        for c, a in enumerate(range(v0, v1, vpc)):
            b = min(a + vpc, v1)
            s = c & 1
            r0, r1 = held_rows(a, b, H)
            # halo carry: the rows this chunk shares with the previous one
            # (its last LOW_HALO rows) are copied device-to-device instead of
            # crossing PCIe again; only rows [h0, r1) come from the host
            carry = 0
            if prev is not None and prev[1] <= r0 < prev[2]:
                carry = prev[2] - r0
            h0 = r0 + carry
            n = (r1 - h0) * row_elems
            if window is None and n:
                if copied[s] is not None:
                    copied[s].synchronize()  # staging[s] uploaded: free again
                _read_parallel(src, h0, r1, staging[s].numpy(), row_elems, pool)
                chunk = staging[s][:n]
            elif n:
                chunk = window(h0, r1).reshape(-1)
            with t.cuda.stream(copy):
                if done[s] is not None:
                    copy.wait_event(done[s])  # dbuf[s] consumed by the previous kernel
                if carry:  # after the previous chunk's upload (same stream)
                    pb, p0, p1 = prev
                    dbuf[s][:carry * row_elems].copy_(dbuf[pb][(r0 - p0) * row_elems:(p1 - p0) * row_elems],
                                                      non_blocking=True)
                if n:
                    dbuf[s][carry * row_elems:carry * row_elems + n].copy_(chunk, non_blocking=True)
                ev = t.cuda.Event()
                ev.record(copy)
                copied[s] = ev
            compute.wait_event(copied[s])
            view = dbuf[s][:(r1 - r0) * row_elems].view((r1 - r0,) + tuple(src.shape[1:]))
            kind.launch(ndim, view, src.shape, M, src.quant, (a, b), first=r0, hist=hist)
            ev = t.cuda.Event()
            ev.record(compute)
            done[s] = ev
            prev = (s, r0, r1)
    finally:
        if pool is not None:
            pool.shutdown(wait=True)
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
