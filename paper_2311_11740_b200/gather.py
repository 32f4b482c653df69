"""Gather drivers: source -> device transition histogram.

Replaces the reference drivers gather_{2d,3d}_{serial,parallel} and their
sliding-window streaming loops (contrib2d.py:235-294, contrib3d.py:392-458,
_parallel.py:8-33) with:

* resident sources (``MemorySource``, ``DeviceSource``): one launch per vertex
  row block on the field already in HBM;
* streamed sources (``ArraySource``, ``BmpSource``, ``RawVolumeSource``):
  chunks of cell rows/planes read into two pinned host buffers and copied to
  two device buffers on a side stream, so the read + H2D of chunk c+1 overlaps
  the kernel on chunk c.  Chunk c covers vertex rows [a, b) and holds cell
  rows [a-1, b-1]; the one-row halo is simply re-read;
* several GPUs in one process (``devices=[...]``): vertex-row slabs per GPU
  like split_blocks, histograms summed after the join.

Every path produces the same histogram bit for bit: integer sums commute.
"""

from __future__ import annotations

import numpy as np

from . import engine
from ._parallel import split_blocks

DEFAULT_CHUNK_BYTES = 256 << 20


def _torch_dtype(np_dtype):
    t = engine.torch()
    return {np.dtype(np.int32): t.int32, np.dtype(np.uint8): t.uint8, np.dtype(np.uint16): t.uint16,
            np.dtype(np.float32): t.float32}[np.dtype(np_dtype)]


def resident_hist(src, ndim, device, rows, workers=1, hist=None):
    x, quant = src.device_field(device)
    if hist is None:
        hist = engine.new_hist(ndim, src.max_level, device)
    v0, v1 = rows
    for a, b in split_blocks(v1 - v0, workers):
        engine.launch_hist(ndim, x, src.shape, src.max_level, quant, rows=(v0 + a, v0 + b), hist=hist)
    return hist


def stream_hist(src, ndim, device, rows, chunk_bytes=DEFAULT_CHUNK_BYTES, hist=None):
    """Double-buffered pinned-host -> HBM streaming of a source's rows/planes."""
    t = engine.torch()
    H = src.height
    M = src.max_level
    row_elems = src.width * (src.depth if ndim == 3 else 1)
    itemsize = np.dtype(src.dtype).itemsize
    tdt = _torch_dtype(src.dtype)
    cap = max(2, int(chunk_bytes // max(1, row_elems * itemsize)))  # cell rows per buffer
    cap = min(cap, H + 1)
    vpc = max(1, cap - 1)  # vertex rows per chunk (one halo row)
    if hist is None:
        hist = engine.new_hist(ndim, M, device)
    pinned = [t.empty(cap * row_elems, dtype=tdt, pin_memory=True) for _ in range(2)]
    dbuf = [t.empty(cap * row_elems, dtype=tdt, device=device) for _ in range(2)]
    src.note_resident(2 * cap * row_elems * itemsize)
    compute = t.cuda.current_stream(device)
    copy = t.cuda.Stream(device)
    copied = [t.cuda.Event() for _ in range(2)]
    done = [None, None]
    v0, v1 = rows
    for c, a in enumerate(range(v0, v1, vpc)):
        b = min(a + vpc, v1)
        s = c & 1
        r0, r1 = max(a - 1, 0), min(b - 1, H - 1) + 1
        n = (r1 - r0) * row_elems
        if done[s] is not None:
            done[s].synchronize()  # pinned[s] / dbuf[s] free again
        src.read_rows(r0, r1, pinned[s].numpy()[:n])
        with t.cuda.stream(copy):
            if done[s] is not None:
                copy.wait_event(done[s])
            dbuf[s][:n].copy_(pinned[s][:n], non_blocking=True)
            copied[s].record(copy)
        compute.wait_event(copied[s])
        view = dbuf[s][:n].view((r1 - r0,) + tuple(src.shape[1:]))
        engine.launch_hist(ndim, view, src.shape, M, src.quant, rows=(a, b), first=r0, hist=hist)
        ev = t.cuda.Event()
        ev.record(compute)
        done[s] = ev
    return hist


def source_hist(src, ndim, device=None, workers=1, rows=None, chunk_bytes=DEFAULT_CHUNK_BYTES):
    """Transition histogram of ``src`` for vertex rows ``rows`` on one GPU."""
    dev = engine.default_device(device)
    rows = rows if rows is not None else (0, src.height + 1)
    if src.mode in ("in-memory", "device"):
        return resident_hist(src, ndim, dev, rows, workers)
    return stream_hist(src, ndim, dev, rows, chunk_bytes)


def multi_device_hist(src, ndim, devices, chunk_bytes=DEFAULT_CHUNK_BYTES):
    """Vertex-row slabs over several GPUs of this process; returns the summed
    histogram on devices[0].  Resident host fields upload only each slab's
    planes plus the one-plane halo."""
    devs = [engine.default_device(d) for d in devices]
    blocks = split_blocks(src.height + 1, len(devs))
    parts = []
    for dev, (a, b) in zip(devs, blocks):
        if src.mode == "in-memory":
            r0, r1 = max(a - 1, 0), min(b - 1, src.height - 1) + 1
            x = engine.to_device(src.field.values[r0:r1], dev)
            h = engine.new_hist(ndim, src.max_level, dev)
            parts.append(engine.launch_hist(ndim, x, src.shape, src.max_level,
                                            engine.QuantSpec.identity(), rows=(a, b), first=r0, hist=h))
        elif src.mode == "device":
            raise ValueError("a DeviceSource lives on one GPU; use devices=None")
        else:
            parts.append(stream_hist(src, ndim, dev, (a, b), chunk_bytes))
    total = parts[0]
    for p in parts[1:]:
        total += p.to(devs[0])
    return total
