"""GPU parity of the drop-in 3D map kernel (ft_hist3d: the register-march
hist3d_march, default; hist3d_pair / hist3d_tiled on FT_MAP3D) against the
pinned oracle, bit-exact maps: row / column extents around the 64-row CTA
tiles and 62-column warp strips (vertex rows 0..W and columns 0..D, halo
halves, guarded boundary strips), plane segments, level counts up to the
kernel's limit."""
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
                                     (2, 130, 64, 1100), (17, 20, 130, 0)])
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
