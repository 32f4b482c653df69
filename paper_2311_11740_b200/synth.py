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


# --------------------------------------------------------------------------
# BASELINE.json configs (shared by bench.py, tools/prof_run.py and the
# config-scale parity tests, tests/test_gpu_configs.py)

CONFIG_NAMES = ("c1", "c2", "c3", "c4a", "c4b", "c5")


def config_field(name, device, seed=2311, planes=None):
    """The synthetic input of BASELINE config ``name`` on ``device``.

    Returns a dict: ``x`` (CUDA tensor: float32 samples, or uint8 / uint16
    raw values), ``M`` (max level), ``value_range`` ((lo, hi) for
    quantize_with_range, or None for identity levels), ``shape`` (the global
    field shape; for C3 the image shape), ``batch`` (images, C3 only).
    ``planes`` = (p0, p1) builds only those planes of the 3D f32 configs
    (bit-identical to the same planes of the whole field; C5 slabs)."""
    import torch

    if name == "c1":  # 256^2 i.i.d. Uniform[0,1), 100 levels on [0, 1]
        g = torch.Generator(device="cpu")
        g.manual_seed(seed)
        x = torch.rand((256, 256), generator=g, dtype=torch.float32).to(device)
        return dict(x=x, M=99, value_range=(0.0, 1.0), shape=(256, 256), batch=1)
    if name == "c2":  # 8192^2 GRF sigma 4 px, min-max to [0, 1], 256 levels
        x = grf_2d((8192, 8192), 4.0, seed, device)
        normalise_(x, x.min(), x.max())
        return dict(x=x, M=255, value_range=(0.0, 1.0), shape=(8192, 8192), batch=1)
    if name == "c3":  # 512 u8 images 1024^2, sigma ~ U[1, 8] px, quantised to 0..255
        n, shape = 512, (1024, 1024)
        sig = np.random.default_rng(seed).uniform(1.0, 8.0, n)
        x = torch.empty((n,) + shape, dtype=torch.uint8, device=device)
        for b in range(n):
            im = grf_2d(shape, float(sig[b]), seed + b, device)
            im = (im - im.min()) / (im.max() - im.min())
            x[b] = torch.floor(im * 255 + 0.5).to(torch.uint8)
        return dict(x=x, M=255, value_range=None, shape=shape, batch=n)
    if name in ("c4a", "c5"):
        shape, sigma, M = {"c4a": ((512, 512, 512), 3.0, 255), "c5": ((2048, 2048, 2048), 4.0, 511)}[name]
        p0, p1 = planes if planes is not None else (0, shape[0])
        x = grf_slab(shape, sigma, seed, (p0, p1), device)
        if planes is None:
            lo, hi = x.min(), x.max()
        else:  # the global extrema (needs the whole field once; cached per process)
            lo, hi = _global_extrema(shape, sigma, seed, device)
        normalise_(x, lo, hi)
        return dict(x=x, M=M, value_range=(0.0, 1.0), shape=shape, batch=1)
    if name == "c4b":  # 1024 x 1024 x 256 u16 cube (sigma 3), quantize(raw, 1023) auto-range
        shape = (1024, 1024, 256)
        x = grf_slab(shape, 3.0, seed, (0, shape[0]), device)
        normalise_(x, x.min(), x.max())
        x = torch.floor(x * 65535 + 0.5).to(torch.int32).to(torch.uint16)
        return dict(x=x, M=1023, value_range="auto", shape=shape, batch=1)
    raise ValueError(f"unknown config {name!r}")


_EXTREMA = {}


def _global_extrema(shape, sigma, seed, device, chunk=256):
    key = (tuple(shape), float(sigma), int(seed))
    if key not in _EXTREMA:
        lo = hi = None
        for p0 in range(0, shape[0], chunk):
            s = grf_slab(shape, sigma, seed, (p0, min(p0 + chunk, shape[0])), device)
            a, b = s.min(), s.max()
            lo = a if lo is None else min(lo, a)
            hi = b if hi is None else max(hi, b)
            del s
        _EXTREMA[key] = (lo, hi)
    return _EXTREMA[key]


class PeriodicPlanes:
    """Streaming source for fields larger than host memory (C5s: 4096^3 f32,
    256 GiB): a (H, W, D) float32 field whose planes repeat with period P,
    plane p = base[p % P], served from a PINNED ring holding the P base planes
    twice, so any window of <= P planes is one contiguous pinned slice the
    streaming engine DMAs from (``pinned_window``).  With a base generated
    periodic along i (``grf_slab`` wraps), the tiled field is a smooth GRF of
    the full size.  Bench / test helper, not part of the reference API."""

    mode = "file-backed"
    ndim = 3
    parallel_reads = True

    def __init__(self, ring, height, max_level, value_range):
        from .quant import QuantSpec

        P2, W, D = ring.shape
        if P2 % 2 or not ring.is_pinned():
            raise ValueError("ring must be a pinned (2P, W, D) tensor")
        self.ring, self.P = ring, P2 // 2
        self.height, self.width, self.depth = int(height), W, D
        self.shape = (self.height, W, D)
        self.dtype = np.dtype(np.float32)
        self.max_level = int(max_level)
        self.quant = QuantSpec.for_range(value_range[0], value_range[1], self.max_level)
        self.peak_field_bytes = ring.numel() * ring.element_size()

    def note_resident(self, nbytes):
        self.peak_field_bytes = max(self.peak_field_bytes, nbytes)

    def pinned_window(self, r0, r1):
        if r1 - r0 > self.P:
            raise ValueError(f"window of {r1 - r0} planes exceeds the ring period {self.P}")
        s = r0 % self.P
        return self.ring[s:s + (r1 - r0)]

    def read_rows(self, r0, r1, out):
        out.reshape(r1 - r0, -1)[:] = self.pinned_window(r0, r1).numpy().reshape(r1 - r0, -1)
