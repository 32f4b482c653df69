"""Config-scale parity: every BASELINE.json config at its full size, the CUDA
path (C ABI) against the CPU oracle, bit for bit.

The north star asks for bit-exact EC / perimeter / area / surface-area /
volume curves on all five configs.  Each test builds the config's seeded
synthetic field on the GPU (``synth.config_field``: shapes, sigmas, level
counts and quantization of BASELINE.json configs[0..4]), copies the same
bytes to the host, runs the oracle (oracle/ft_oracle.c, the C restatement of
contrib2d.py:161-294 / contrib3d.py:241-458 and fields.py:20-45, all host
threads) and compares

* the contribution maps of the drop-in ``gather_*`` path (q_in / q_out), and
* every curve of the fused ``descriptor_curves`` path (line-decomposition /
  lattice kernels) and of ``descriptor_curve`` on the maps

against the oracle's maps and ``eighths @ counts_at_levels`` (descriptors.py:
153-178).  C5 (2048^3, 32 GiB) is checked over the WHOLE field: the oracle
runs slab by slab (vertex rows [a, b) need cell planes a-1 .. b-1) and its
maps are summed -- integer sums commute, so the sum is the whole-field map.
This mirrors the reference's acceptance c5 (pkg/tests/test_acceptance.py:
288-304: in-memory vs partitioned gathers are identical) at config size.
"""
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

THREADS = os.cpu_count() or 1
T2D = (("ec", "8C"), ("ec", "4C"), ("perimeter", "8C"), ("area", "8C"))
T3D = ("ec", "surface-area", "volume", "perimeter")


@pytest.fixture(scope="module")
def ft():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_11740_b200 as ft
    return ft


def _dev():
    import torch
    return torch.device("cuda", 0)


def _check_maps(cmap, q_in, q_out, what):
    assert np.array_equal(cmap.q_in, q_in), f"{what}: q_in differs from the oracle"
    assert np.array_equal(cmap.q_out, q_out), f"{what}: q_out differs from the oracle"


def _check_curves(ft, orc, curves, tables, q_in, q_out, M, what):
    for c, t in zip(curves, tables):
        ref = orc.descriptor_numerators(q_in, q_out, M, t.eighths)
        assert np.array_equal(c.numerators, ref), f"{what}: {t.descriptor} curve differs from the oracle"


def _tables_2d(ft):
    return [ft.builtin_weights(*t) for t in T2D]


def _tables_3d(ft):
    return [ft.builtin_weights(d, "26C") for d in T3D]


def test_config2_8192sq_f32(ft, orc):
    from paper_2311_11740_b200 import synth
    cfg = synth.config_field("c2", _dev())
    x, M = cfg["x"], cfg["M"]
    xh = x.cpu().numpy()
    q_in, q_out = orc.gather2d(xh, M, value_range=(0.0, 1.0), workers=THREADS)
    src = ft.DeviceSource(x, M, value_range=(0.0, 1.0))
    cmap = ft.gather_2d_serial(src)
    _check_maps(cmap, q_in, q_out, "C2 map")
    tabs = _tables_2d(ft)
    _check_curves(ft, orc, ft.descriptor_curves(src, tabs), tabs, q_in, q_out, M, "C2 fused")
    _check_curves(ft, orc, [ft.descriptor_curve(cmap, t) for t in tabs], tabs, q_in, q_out, M, "C2 map curves")
    # the low-memory (streamed from host) path on the same bytes
    _check_curves(ft, orc, ft.descriptor_curves(ft.ArraySource(xh, M, value_range=(0.0, 1.0)), tabs,
                                                chunk_bytes=37 << 20), tabs, q_in, q_out, M, "C2 streamed")


def test_config3_512_u8_images(ft, orc):
    from paper_2311_11740_b200 import synth
    cfg = synth.config_field("c3", _dev())
    x, M, n = cfg["x"], cfg["M"], cfg["batch"]
    xh = x.cpu().numpy()
    tabs = _tables_2d(ft)
    maps = ft.gather_2d_batch(x, M)
    curves = ft.descriptor_curves_batch(x, M, tabs)
    ec_only = ft.descriptor_curves_batch(x, M, tabs[:1])  # the per-image EC curve (line kernel)
    assert len(maps) == len(curves) == n
    for b in range(n):
        q_in, q_out = orc.gather2d(xh[b], M, workers=THREADS)
        _check_maps(maps[b], q_in, q_out, f"C3 image {b} map")
        _check_curves(ft, orc, curves[b], tabs, q_in, q_out, M, f"C3 image {b}")
        _check_curves(ft, orc, ec_only[b], tabs[:1], q_in, q_out, M, f"C3 image {b} EC")


def test_config4a_512cube_f32(ft, orc):
    from paper_2311_11740_b200 import synth
    cfg = synth.config_field("c4a", _dev())
    x, M = cfg["x"], cfg["M"]
    q_in, q_out = orc.gather3d(x.cpu().numpy(), M, value_range=(0.0, 1.0), workers=THREADS)
    src = ft.DeviceSource(x, M, value_range=(0.0, 1.0))
    cmap = ft.gather_3d_serial(src)
    _check_maps(cmap, q_in, q_out, "C4a map")
    tabs = _tables_3d(ft)
    _check_curves(ft, orc, ft.descriptor_curves(src, tabs[:3], path="lines"), tabs[:3], q_in, q_out, M,
                  "C4a lines")
    _check_curves(ft, orc, ft.descriptor_curves(src, tabs), tabs, q_in, q_out, M, "C4a fused (+perimeter)")
    _check_curves(ft, orc, [ft.descriptor_curve(cmap, t) for t in tabs], tabs, q_in, q_out, M, "C4a map curves")
    assert ft.gather_3d_parallel(src, 7) == cmap


def test_config4b_u16_cube_auto_range(ft, orc, tmp_path):
    from paper_2311_11740_b200 import engine, synth
    cfg = synth.config_field("c4b", _dev())
    x, M = cfg["x"], cfg["M"]
    raw = x.cpu().numpy()
    # the reference's quantize(raw, 1023): range = the data's own min / max
    lo, hi = engine.minmax_device(x)
    assert (lo, hi) == (float(raw.min()), float(raw.max()))
    levels = orc.quantize(raw, M)
    q_in, q_out = orc.gather3d(levels, M, workers=THREADS)
    src = ft.DeviceSource(x, M, value_range=(lo, hi))
    cmap = ft.gather_3d_serial(src)
    _check_maps(cmap, q_in, q_out, "C4b map")
    tabs = _tables_3d(ft)
    _check_curves(ft, orc, ft.descriptor_curves(src, tabs), tabs, q_in, q_out, M, "C4b fused")
    # as a user of the reference gets there: a raw u16 file (h=1024, w=1024, d=256)
    path = tmp_path / "c4b.raw"
    raw.tofile(path)
    dims = (raw.shape[1], raw.shape[0], raw.shape[2])
    assert np.array_equal(ft.read_raw_volume(path, dims, "u16", M).values, levels)
    with ft.open_raw_lowmem(path, dims, "u16", M) as lowmem:
        assert lowmem.value_range == (lo, hi)
        _check_maps(ft.gather_3d_serial(lowmem), q_in, q_out, "C4b low-memory map")
        _check_curves(ft, orc, ft.descriptor_curves(lowmem, tabs[:3]), tabs[:3], q_in, q_out, M,
                      "C4b low-memory curves")


def test_config5_2048cube_f32_whole_field(ft, orc):
    import torch

    from paper_2311_11740_b200 import synth
    from paper_2311_11740_b200._parallel import split_blocks
    cfg = synth.config_field("c5", _dev())
    x, M = cfg["x"], cfg["M"]
    H = x.shape[0]
    src = ft.DeviceSource(x, M, value_range=(0.0, 1.0))
    tabs = _tables_3d(ft)
    fused = ft.descriptor_curves(src, tabs[:3])  # ft_lines3d: the benchmark kernel
    cmap = ft.gather_3d_serial(src)              # hist3d_march: the drop-in map kernel
    torch.cuda.synchronize()
    # whole-field oracle, slab by slab (about 1 minute on 16 host threads)
    q_in = np.zeros((21, M + 2), np.uint64)
    q_out = np.zeros_like(q_in)
    for a, b in split_blocks(H + 1, 16):
        r0, r1 = max(a - 1, 0), min(b, H)
        slab = x[r0:r1].cpu().numpy()
        qi, qo = orc.gather3d(slab, M, value_range=(0.0, 1.0), workers=THREADS, rows=(a - r0, b - r0))
        q_in += qi
        q_out += qo
    _check_maps(cmap, q_in, q_out, "C5 map")
    _check_curves(ft, orc, fused, tabs[:3], q_in, q_out, M, "C5 lines")
    _check_curves(ft, orc, [ft.descriptor_curve(cmap, t) for t in tabs], tabs, q_in, q_out, M, "C5 map curves")
