"""Seeded synthetic fields for benchmarks and large-size tests (BASELINE.json
configs).  No dataset ships with the reference; these stand in with the
configs' shapes and value distributions.

Gaussian random fields are built slab-locally so every z-slab partition sees
bit-identical bytes: white noise is drawn per plane from a generator seeded by
(seed, plane index), smoothed with a truncated (4 sigma) Gaussian with
periodic ("wrap") boundaries by a fixed sequence of elementwise
multiply-adds -- deterministic and independent of how planes are grouped --
then min-max normalised to [0, 1] with the global extrema.
"""

from __future__ import annotations

import math

import numpy as np


def gaussian_taps(sigma):
    r = int(math.ceil(4 * sigma))
    t = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-t * t / (2 * sigma * sigma))
    return (w / w.sum()).astype(np.float32), r


def _plane_noise(torch, seed, p, shape, device):
    g = torch.Generator(device=device)
    g.manual_seed((int(seed) * 1_000_003 + int(p)) & 0x7FFFFFFFFFFFFFFF)
    return torch.randn(shape, generator=g, device=device, dtype=torch.float32)


def _smooth_axis_(torch, x, w, r, dim, out):
    """out = sum_t w[t] * roll(x, t - r, dim) with wrap, in a fixed order."""
    n = x.shape[dim]
    out.zero_()
    for ti, wt in enumerate(w.tolist()):
        s = (ti - r) % n  # out[i] += w * x[i - (ti - r)]  (circular)
        if s == 0:
            out.add_(x, alpha=wt)
            continue
        out.narrow(dim, s, n - s).add_(x.narrow(dim, 0, n - s), alpha=wt)
        out.narrow(dim, 0, s).add_(x.narrow(dim, n - s, s), alpha=wt)
    return out


def grf_slab(shape, sigma, seed, planes, device, chunk=32):
    """Un-normalised smoothed white noise for global planes [p0, p1) of a
    periodic 3D field of ``shape`` (H, W, D); float32 CUDA tensor."""
    import torch

    H, W, D = shape
    p0, p1 = planes
    w, r = gaussian_taps(sigma)
    r_i = min(r, (H - 1) // 2) if H > 1 else 0
    lo, hi = p0 - r_i, p1 + r_i
    # 1) in-plane smoothing (k, then j) of every plane in [lo, hi)
    inplane = torch.empty((hi - lo, W, D), dtype=torch.float32, device=device)
    tmp = torch.empty((chunk, W, D), dtype=torch.float32, device=device)
    for c0 in range(lo, hi, chunk):
        c1 = min(c0 + chunk, hi)
        blk = torch.stack([_plane_noise(torch, seed, p % H, (W, D), device) for p in range(c0, c1)])
        t = tmp[: c1 - c0]
        _smooth_axis_(torch, blk, w, min(r, (D - 1) // 2), 2, t)
        _smooth_axis_(torch, t, w, min(r, (W - 1) // 2), 1, inplane[c0 - lo:c1 - lo])
        del blk
    del tmp
    # 2) smoothing along i (planes), periodic through the drawn margins
    out = torch.zeros((p1 - p0, W, D), dtype=torch.float32, device=device)
    wi, _ = gaussian_taps(sigma)
    wi = wi[r - r_i: r + r_i + 1] if r_i < r else wi
    for ti, wt in enumerate(wi.tolist()):
        out.add_(inplane[ti: ti + (p1 - p0)], alpha=wt)
    del inplane
    return out


def normalise_(x, lo, hi):
    """(x - lo) / (hi - lo) in float32, in place."""
    x.sub_(lo).div_(hi - lo)
    return x


def grf_2d(shape, sigma, seed, device):
    """2D smoothed Gaussian random field (periodic), un-normalised."""
    import torch

    H, W = shape
    w, r = gaussian_taps(sigma)
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    x = torch.randn((H, W), generator=g, device=device, dtype=torch.float32)
    t = torch.empty_like(x)
    _smooth_axis_(torch, x, w, min(r, (W - 1) // 2), 1, t)
    _smooth_axis_(torch, t, w, min(r, (H - 1) // 2), 0, x)
    return x
