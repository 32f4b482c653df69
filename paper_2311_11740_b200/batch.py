"""Batched 2D API (BASELINE config 3: 512 images of 1024^2, per-image curves).

The reference has no batch call -- the paper dispatches many small images in
parallel and a user loops ``gather_2d_*`` over images.  Here a
stack of equally shaped images is one launch: every CTA work item belongs to
one image and flushes into that image's histogram (csrc ft_hist2d /
ft_lattice2d ``batch``), so the per-image maps and curves equal the
per-image reference results exactly.
"""

from __future__ import annotations

import numpy as np

from . import engine, lattice
from .contrib2d import ContributionMap2D
from .descriptors import DescriptorCurve
from .quant import QuantSpec


def _stack(images, device):
    t = engine.torch()
    if isinstance(images, t.Tensor) and images.is_cuda:
        x = images.contiguous()
    else:
        x = engine.to_device(images, device)
    if x.dim() != 3:
        raise ValueError("expected a stack of 2D images (N, H, W)")
    return x


def _quant(x, max_level, value_range):
    t = engine.torch()
    if value_range is not None:
        return QuantSpec.for_range(value_range[0], value_range[1], max_level)
    if x.dtype == t.float32:
        raise ValueError("float32 images need value_range=(lo, hi)")
    return QuantSpec.identity()


def gather_2d_batch(images, max_level, value_range=None, device=None):
    """Contribution maps of every image of an (N, H, W) stack (int32 levels,
    uint8/uint16 levels, or raw samples with ``value_range``)."""
    dev = engine.default_device(device)
    x = _stack(images, dev)
    N, H, W = x.shape
    M = int(max_level)
    hist = engine.launch_hist(2, x, (H, W), M, _quant(x, M, value_range), rows=(0, H + 1), batch=N,
                              batch_stride=H * W)
    q_in, q_out, _ = engine.finalize(2, M, hist.view(N, 6, M + 2), maps=True)
    qi, qo = engine.as_uint64(q_in), engine.as_uint64(q_out)
    return [ContributionMap2D(W, H, M, qi[b], qo[b]) for b in range(N)]


def descriptor_curves_batch(images, max_level, tables, value_range=None, device=None):
    """Per-image DescriptorCurves ([image][table]) of an (N, H, W) stack,
    fused on the GPU (lattice kernel when every table is in its span)."""
    dev = engine.default_device(device)
    x = _stack(images, dev)
    N, H, W = x.shape
    M = int(max_level)
    tables = list(tables)
    if any(t.dimension != 2 for t in tables):
        raise ValueError("batched curves take 2D weight tables")
    quant = _quant(x, M, value_range)
    rw = [lattice.row_weights(2, tuple(int(e) for e in t.eighths)) for t in tables]
    if all(r is not None for r in rw) and engine.lattice_ok(2, (H, W), M):
        maxes = any(lattice.needs_max_rows(r[0]) for r in rw)
        hist = engine.new_lattice_hist(2, M, dev, batch=N).view(N, 4, M + 2)  # batch axis kept for N == 1
        engine.launch_lattice(2, x, (H, W), M, quant, rows=(0, H + 1), hist=hist, batch=N, batch_stride=H * W,
                              maxes=maxes)
        num = engine.curves_from_rows(hist, M, np.array([r[0] for r in rw])).cpu().numpy()
        num = num // np.array([r[1] for r in rw])[None, :, None]
    else:
        hist = engine.launch_hist(2, x, (H, W), M, quant, rows=(0, H + 1), batch=N, batch_stride=H * W)
        _, _, num = engine.finalize(2, M, hist.view(N, 6, M + 2), maps=False, tables=[t.eighths for t in tables])
        num = num.cpu().numpy()
    return [[DescriptorCurve(t.descriptor, t.connectivity, M, num[b, i]) for i, t in enumerate(tables)]
            for b in range(N)]
