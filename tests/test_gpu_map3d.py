"""GPU parity of the drop-in 3D map kernels (ft_hist3d: the register-march
hist3d_march up to M ~ 1150, hist3d_wide beyond) against the pinned oracle,
bit-exact maps: row / column extents around the 64-row CTA tiles and
62-column warp strips (vertex rows 0..W and columns 0..D, halo halves,
guarded boundary strips), plane segments, level counts on both sides of the
march kernel's limit up to u16 identity levels (M = 65535)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ft():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_11740_b200 as ft
    return ft


@pytest.mark.parametrize("H,W,D,M", [(1, 1, 1, 3), (2, 1, 61, 7), (3, 63, 62, 255), (5, 64, 63, 15),
                                     (4, 65, 124, 255), (6, 67, 125, 1), (3, 128, 187, 511), (9, 3, 2, 1000),
                                     (2, 130, 64, 1100), (17, 20, 130, 0),
                                     (5, 9, 13, 1200), (4, 70, 67, 4095), (3, 11, 130, 65535)])
def test_map3d_vs_oracle(ft, orc, H, W, D, M):
    lv = np.random.default_rng(H * 10007 + W * 101 + D).integers(0, M + 1, size=(H, W, D), dtype=np.int32)
    m = ft.gather_3d_serial(ft.Field3D(lv, M))
    q_in, q_out = orc.gather3d(lv, M, workers=8)
    assert np.array_equal(m.q_in, q_in) and np.array_equal(m.q_out, q_out)


def test_map3d_smooth_f32_workers_and_streaming(ft, orc):
    import torch
    from scipy.ndimage import gaussian_filter
    x = gaussian_filter(np.random.default_rng(8).standard_normal((40, 70, 131)).astype(np.float32), 2.0, mode="wrap")
    x = ((x - x.min()) / (x.max() - x.min())).astype(np.float32)
    q_in, q_out = orc.gather3d(x, 255, value_range=(0.0, 1.0), workers=8)
    src = ft.DeviceSource(torch.from_numpy(x).cuda(), 255, value_range=(0.0, 1.0))
    for workers in (1, 3):
        m = ft.gather_3d_parallel(src, workers)
        assert np.array_equal(m.q_in, q_in) and np.array_equal(m.q_out, q_out), workers
    m = ft.gather_3d_serial(ft.ArraySource(x, 255, value_range=(0.0, 1.0)))  # streamed windows
    assert np.array_equal(m.q_in, q_in) and np.array_equal(m.q_out, q_out)


def test_map3d_u16_4095_raw_and_curves(ft, orc, tmp_path):
    """read_raw_volume(..., "u16", 4095) -> gather_3d_serial and the fused
    curves at M = 4095 (reference sources.py:247-269 accepts any max_level;
    contrib3d.py:417-419 allocates (21, M + 2) with no limit)."""
    vol = np.random.default_rng(9).integers(0, 65536, size=(6, 40, 70)).astype(np.uint16)
    p = tmp_path / "v.raw"
    vol.tofile(p)
    dims = (40, 6, 70)
    levels = orc.quantize(vol, 4095)
    q_in, q_out = orc.gather3d(levels, 4095, workers=8)
    f = ft.read_raw_volume(p, dims, "u16", 4095)
    assert np.array_equal(f.values, levels)
    m = ft.gather_3d_serial(f)
    assert np.array_equal(m.q_in, q_in) and np.array_equal(m.q_out, q_out)
    with ft.open_raw_lowmem(p, dims, "u16", 4095) as src:
        m2 = ft.gather_3d_serial(src)
        assert np.array_equal(m2.q_in, q_in) and np.array_equal(m2.q_out, q_out)
    tabs = [ft.builtin_weights(d, "26C") for d in ("ec", "perimeter", "surface-area", "volume")]
    for path in ("auto", "map"):
        for c, t in zip(ft.descriptor_curves(f, tabs, path=path), tabs):
            assert np.array_equal(c.numerators, orc.descriptor_numerators(q_in, q_out, 4095, t.eighths)), path


def test_map3d_u16_identity_65535(ft, orc):
    import torch
    vol = np.random.default_rng(10).integers(0, 65536, size=(7, 9, 33)).astype(np.uint16)
    q_in, q_out = orc.gather3d(vol, 65535, workers=8)
    src = ft.DeviceSource(torch.from_numpy(vol.astype(np.int32)).to(torch.uint16).cuda(), 65535)
    m = ft.gather_3d_serial(src)
    assert np.array_equal(m.q_in, q_in) and np.array_equal(m.q_out, q_out)
    tabs = [ft.builtin_weights(d, "26C") for d in ("ec", "surface-area", "volume")]
    for c, t in zip(ft.descriptor_curves(src, tabs), tabs):
        assert np.array_equal(c.numerators, orc.descriptor_numerators(q_in, q_out, 65535, t.eighths))
