"""GPU parity of the drop-in 2D map kernels (ft_hist2d: the register-march
hist2d_march, M <= ~7260, and hist2d_wide beyond) against the pinned oracle,
bit-exact maps: widths around the 62-column strip tiling (vertex columns
0..W, halo halves, clamped boundary tiles), level counts up to and past the
march kernel's shared-memory limit up to u16 identity levels (M = 65535),
batches with odd strides."""
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


@pytest.mark.parametrize("H,W,M", [(1, 1, 3), (3, 2, 0), (7, 61, 255), (40, 62, 15), (33, 63, 255), (9, 64, 255),
                                   (70, 123, 511), (65, 124, 7), (64, 125, 255), (5, 126, 2000), (130, 187, 255),
                                   (31, 250, 7000), (12, 77, 8000), (9, 130, 65535), (3, 2, 100000)])
def test_map2d_vs_oracle(ft, orc, H, W, M):
    lv = np.random.default_rng(H * 7919 + W).integers(0, M + 1, size=(H, W), dtype=np.int32)
    m = ft.gather_2d_serial(ft.Field2D(lv, M))
    q_in, q_out = orc.gather2d(lv, M)
    assert np.array_equal(m.q_in, q_in) and np.array_equal(m.q_out, q_out)


@pytest.mark.parametrize("workers", [1, 3])
def test_map2d_smooth_f32_and_workers(ft, orc, workers):
    import torch
    from scipy.ndimage import gaussian_filter
    x = gaussian_filter(np.random.default_rng(2).standard_normal((190, 311)).astype(np.float32), 2.5, mode="wrap")
    x = ((x - x.min()) / (x.max() - x.min())).astype(np.float32)
    src = ft.DeviceSource(torch.from_numpy(x).cuda(), 255, value_range=(0.0, 1.0))
    m = ft.gather_2d_parallel(src, workers)
    q_in, q_out = orc.gather2d(x, 255, value_range=(0.0, 1.0))
    assert np.array_equal(m.q_in, q_in) and np.array_equal(m.q_out, q_out)


def test_map2d_batch_odd_width(ft, orc):
    imgs = np.random.default_rng(4).integers(0, 256, size=(9, 37, 71), dtype=np.uint8)
    maps = ft.gather_2d_batch(imgs, 255)
    for b in (0, 4, 8):
        q_in, q_out = orc.gather2d(imgs[b], 255)
        assert np.array_equal(maps[b].q_in, q_in) and np.array_equal(maps[b].q_out, q_out), b


def test_map2d_large_levels_batch_and_curves(ft, orc):
    """u16 identity levels (M = 65535) through the batch API and the fused
    curves: the wide map kernel + device finalize, any level count."""
    imgs = np.random.default_rng(6).integers(0, 65536, size=(3, 29, 41)).astype(np.uint16)
    maps = ft.gather_2d_batch(imgs, 65535)
    tabs = [ft.builtin_weights(*t) for t in (("ec", "8C"), ("ec", "4C"), ("perimeter", "8C"), ("area", "8C"))]
    curves = ft.descriptor_curves_batch(imgs, 65535, tabs)
    for b in range(3):
        q_in, q_out = orc.gather2d(imgs[b], 65535)
        assert np.array_equal(maps[b].q_in, q_in) and np.array_equal(maps[b].q_out, q_out), b
        for c, t in zip(curves[b], tabs):
            assert np.array_equal(c.numerators, orc.descriptor_numerators(q_in, q_out, 65535, t.eighths)), b
