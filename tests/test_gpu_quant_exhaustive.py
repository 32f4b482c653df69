"""Exhaustive check of the device quantizers against the reference formula
(fields.py:20-33: clip(floor((x - lo) * M / (hi - lo) + 0.5), 0, M) in
float64) -- every input value, not a sample.

The fused kernels inline three quantizers (include/fieldtopo_b200.h
ft_quantize_probe): to_level (map kernels), to_level4 (march / lattice
kernels; table-free for lo = 0, hi = 2^p) and pack_pow2_sat (line kernels:
FMUL.SAT + FFMA2.RM + FADD2.RM magic floor, the C2 / C4a / C5 path).  Each
runs over ALL float32 bit patterns of the tested window (about 1.07e9 values
for [0, hi] plus the saturating region above and a strided sweep of the
negatives) and over all 65536 uint16 values, and must equal the float64
reference evaluated on the GPU (IEEE-exact double add / mul / div, the same
operation order as numpy).  Tolerance: none (integer levels)."""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CHUNK = 1 << 28


@pytest.fixture(scope="module")
def ft():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_11740_b200 as ft
    return ft


def _probe(x, spec, M, path):
    import ctypes

    import torch

    from paper_2311_11740_b200 import _lib, engine
    from paper_2311_11740_b200.quant import device_struct
    out = torch.empty(x.numel(), dtype=torch.int32, device=x.device)
    qs, keep = device_struct(spec, x.device)
    rc = _lib.load().ft_quantize_probe(ctypes.c_void_p(x.data_ptr()), engine.dtype_code(x), x.numel(),
                                       ctypes.byref(qs), M, path, ctypes.c_void_p(out.data_ptr()),
                                       engine._stream_ptr(x.device))
    del keep
    _lib.check(rc, "ft_quantize_probe")
    return out


def _reference(x, lo, hi, M):
    import torch
    xd = x.double()
    return torch.clamp(torch.floor((xd - lo) * float(M) / (hi - lo) + 0.5), 0, M).to(torch.int32)


def _bit_windows(a_bits, b_bits, step=1):
    """float32 values whose bit patterns (as int64 of the uint32 pattern) run
    over [a_bits, b_bits) with ``step``, in chunks."""
    import torch
    for s in range(a_bits, b_bits, CHUNK * step):
        e = min(s + CHUNK * step, b_bits)
        u = torch.arange(s, e, step, dtype=torch.int64, device="cuda")
        yield (u - (1 << 32) * (u >= (1 << 31))).to(torch.int32).view(torch.float32)


def _bits(f):
    return int(np.array(f, np.float32).view(np.uint32))


def _check_window(ft, lo, hi, M, paths, windows):
    import torch
    spec = ft.quant.QuantSpec.for_range(lo, hi, M)
    checked = 0
    for a, b, step in windows:
        for x in _bit_windows(a, b, step):
            if x.numel() % 2:
                x = x[:-1]
            ref = _reference(x, lo, hi, M)
            for p in paths:
                got = _probe(x, spec, M, p)
                bad = torch.nonzero(got != ref)
                assert bad.numel() == 0, (lo, hi, M, p, float(x[bad[0, 0]]), int(got[bad[0, 0]]), int(ref[bad[0, 0]]))
            checked += x.numel()
    return spec, checked


@pytest.mark.parametrize("hi,M", [(1.0, 99), (1.0, 255), (1.0, 511), (1.0, 1023), (2.0, 511), (16.0, 255),
                                  (0.125, 511)])
def test_pow2_range_every_float(ft, hi, M):
    """lo = 0, hi = 2^p (the benchmark configs' quantize_with_range(x, 0, 1, M)):
    every float32 in [0, 2 hi), every 61st negative float down to -2 hi."""
    from paper_2311_11740_b200 import _lib, engine
    paths = (0, 1, 2) if engine.lines_ok(M) else (0, 1)
    windows = [(0, _bits(2 * hi), 1), (_bits(-0.0), _bits(-2 * hi), 61)]
    spec, n = _check_window(ft, 0.0, hi, M, paths, windows)
    assert spec.mode == _lib.FT_Q_POW2
    assert n > 1_000_000_000


def test_table_range_every_float(ft):
    """A non-power-of-two range (threshold-table quantizer): every float32 in
    [-4, 13] against quantize_with_range(x, -3.7, 12.1, 255)."""
    windows = [(0, _bits(13.0), 1), (_bits(-0.0), _bits(-4.0), 1)]
    _, n = _check_window(ft, -3.7, 12.1, 255, (0, 1), windows)
    assert n > 2_000_000_000


@pytest.mark.parametrize("lo,hi,M", [(0.0, 65535.0, 1023), (37.0, 65501.0, 1023), (100.0, 60000.0, 4095),
                                     (60000.0, 100.0, 255), (0.0, 65536.0, 511)])
def test_u16_every_value(ft, lo, hi, M):
    """All 65536 uint16 values (C4b: quantize(raw, 1023) on a u16 cube; a
    reversed range takes the walking table)."""
    import torch
    x = torch.arange(65536, dtype=torch.int32, device="cuda").to(torch.uint16)
    spec = ft.quant.QuantSpec.for_range(lo, hi, M)
    ref = _reference(x.to(torch.float32), lo, hi, M)
    for p in (0, 1):
        assert torch.equal(_probe(x, spec, M, p), ref), (lo, hi, M, p)
    # path 3: the line kernels' exact integer decoding of uint16 pairs, taken
    # for increasing integer ranges inside the type; other ranges are refused
    # there (the kernels keep the table for them)
    if lo < hi <= 65535:
        assert torch.equal(_probe(x, spec, M, 3), ref), (lo, hi, M, 3)
    else:
        with pytest.raises(ValueError):
            _probe(x, spec, M, 3)


@pytest.mark.parametrize("lo,hi,M", [(0, 1, 1), (5, 6, 3), (12, 4000, 1023), (1000, 1001, 4095), (0, 65535, 16383),
                                     (1, 65534, 2047), (0, 255, 255), (3, 250, 100), (32768, 32769, 7),
                                     (0, 65535, 1), (17, 40001, 1000)])
def test_u16_integer_decoding_every_value(ft, lo, hi, M):
    """FT_Q_UMAGIC on all 65536 uint16 values for narrow, wide, odd and
    extreme integer ranges against the float64 formula (fields.py:20-33)."""
    import torch
    x = torch.arange(65536, dtype=torch.int32, device="cuda").to(torch.uint16)
    spec = ft.quant.QuantSpec.for_range(float(lo), float(hi), M)
    ref = _reference(x.to(torch.float32), float(lo), float(hi), M)
    assert torch.equal(_probe(x, spec, M, 3), ref), (lo, hi, M)
