"""GPU parity of the 2D line-decomposition curve kernel (ft_lines2d: EC_8C,
perimeter, area; the default fused 2D path when no table needs vertex maxes)
against the reference golden curves, the pinned oracle and ft_lattice2d,
bit-exact: golden fields, random levels with widths around the 62-column
strip tiling, every input dtype / quantizer, batches, streaming windows."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
T2L = (("ec", "8C"), ("perimeter", "8C"), ("area", "8C"))


@pytest.fixture(scope="module")
def ft():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_11740_b200 as ft
    return ft


def _tabs(ft):
    return [ft.builtin_weights(*t) for t in T2L]


def _want(orc, ft, x, M, vr=None):
    q_in, q_out = orc.gather2d(x, M, value_range=vr)
    return [orc.descriptor_numerators(q_in, q_out, M, t.eighths) for t in _tabs(ft)]


def _rows(ft, lv, M):
    import torch
    from paper_2311_11740_b200 import engine
    x = torch.from_numpy(np.ascontiguousarray(lv, np.int32)).cuda()
    return engine.launch_lattice(2, x, lv.shape, M, ft.quant.QuantSpec.identity(), kernel="lines")


def _plan(ft):
    from paper_2311_11740_b200 import lattice
    return lattice.fused_plan(2, [t.eighths for t in _tabs(ft)])


def test_lines2d_golden(ft, golden):
    from paper_2311_11740_b200 import engine, lattice
    assert lattice.fused_plan(2, [t.eighths for t in _tabs(ft)])[1] is False  # no maxes: ft_lines2d
    for n in range(int(golden["n_f2d"])):
        lv, M = golden[f"f2d{n}_levels"], int(golden[f"f2d{n}_M"])
        curves = ft.descriptor_curves(ft.Field2D(lv, M), _tabs(ft), path="lattice")
        for c, t in zip(curves, (0, 2, 3)):
            assert np.array_equal(c.numerators, golden[f"f2d{n}_curves"][t]), (n, t)
        plan = _plan(ft)
        got = engine.curves_from_rows(_rows(ft, lv, M), M, plan[2]).cpu().numpy() // plan[3][:, None]
        for c, t in zip(got, (0, 2, 3)):
            assert np.array_equal(c, golden[f"f2d{n}_curves"][t]), (n, t)


@pytest.mark.parametrize("H,W,M", [(1, 1, 3), (1, 9, 2), (9, 1, 5), (5, 61, 255), (40, 62, 255), (33, 63, 63),
                                   (70, 123, 511), (64, 124, 7), (65, 125, 255), (3, 186, 1000),
                                   (130, 187, 255), (257, 256, 255), (31, 1024, 255), (300, 190, 0)])
def test_lines2d_rows_equal_lattice(ft, H, W, M):
    """ft_lines2d rows (C, E, V) == ft_lattice2d rows, random levels."""
    import torch
    from paper_2311_11740_b200 import engine
    lv = np.random.default_rng(H * 1000 + W).integers(0, M + 1, size=(H, W), dtype=np.int32)
    x = torch.from_numpy(lv).cuda()
    q = ft.quant.QuantSpec.identity()
    a = engine.launch_lattice(2, x, (H, W), M, q, kernel="lines")
    b = engine.launch_lattice(2, x, (H, W), M, q, kernel="lattice")
    assert torch.equal(a[:3, :M + 1], b[:3, :M + 1])  # the sentinel bin M+1 is never read


@pytest.mark.parametrize("dtype,vr,M", [(np.float32, (0.0, 1.0), 255), (np.float32, (0.1, 0.9), 511),
                                        (np.uint16, (0.0, 65535.0), 1000), (np.uint8, None, 255),
                                        (np.uint8, (0.0, 255.0), 99)])
def test_lines2d_dtypes(ft, orc, dtype, vr, M):
    import torch
    from scipy.ndimage import gaussian_filter
    x = gaussian_filter(np.random.default_rng(5).standard_normal((300, 410)).astype(np.float32), 3.0, mode="wrap")
    x = (x - x.min()) / (x.max() - x.min())
    if dtype == np.uint16:
        x = np.floor(x * 65535 + 0.5).astype(np.uint16)
    elif dtype == np.uint8:
        x = np.floor(x * 255 + 0.5).astype(np.uint8)
    else:
        x[7, 9], x[100, 200] = -2.0, 5.0  # out of range: level 0 / M like the reference
    src = ft.DeviceSource(torch.from_numpy(x).cuda(), M, value_range=vr)
    got = ft.descriptor_curves(src, _tabs(ft))
    for c, w in zip(got, _want(orc, ft, x, M, vr)):
        assert np.array_equal(c.numerators, w)


def test_lines2d_batch(ft, orc):
    rng = np.random.default_rng(11)
    imgs = rng.integers(0, 256, size=(37, 70, 131), dtype=np.uint8)
    got = ft.descriptor_curves_batch(imgs, 255, _tabs(ft))
    for b in (0, 1, 17, 36):
        for c, w in zip(got[b], _want(orc, ft, imgs[b], 255)):
            assert np.array_equal(c.numerators, w), b


def test_lines2d_streaming_and_workers(ft, orc):
    from scipy.ndimage import gaussian_filter
    x = gaussian_filter(np.random.default_rng(3).standard_normal((211, 300)).astype(np.float32), 2.0, mode="wrap")
    x = ((x - x.min()) / (x.max() - x.min())).astype(np.float32)
    want = _want(orc, ft, x, 255, (0.0, 1.0))
    for chunk in (3 * 300 * 4, 17 * 300 * 4):
        got = ft.descriptor_curves(ft.ArraySource(x, 255, value_range=(0.0, 1.0)), _tabs(ft), chunk_bytes=chunk)
        assert all(np.array_equal(c.numerators, w) for c, w in zip(got, want)), chunk
    import torch
    src = ft.DeviceSource(torch.from_numpy(x).cuda(), 255, value_range=(0.0, 1.0))
    for workers in (1, 3):
        got = ft.descriptor_curves(src, _tabs(ft), workers=workers)
        assert all(np.array_equal(c.numerators, w) for c, w in zip(got, want)), workers


@pytest.mark.parametrize("H,W,vr,M,batch", [(97, 8192, (0.0, 1.0), 255, 1), (5, 8192, (0.0, 1.0), 511, 1),
                                           (200, 1024, (0.0, 1.0), 255, 1), (1, 1024, (0.0, 2.0), 99, 1),
                                           (33, 1024, (0.0, 1.0), 255, 6)])
def test_lines2d_stride_specialised_f32(ft, orc, H, W, vr, M, batch):
    """The compiled-stride kernels (W = 8192 / 1024, f32 power-of-two range;
    ft_lines2d.cu) on small heights: single images, a batch, row windows of
    a streamed source -- against the oracle."""
    import torch
    from scipy.ndimage import gaussian_filter
    rng = np.random.default_rng(H + W + batch)
    x = gaussian_filter(rng.standard_normal((batch, H, W)).astype(np.float32), (0, 2.0, 2.0), mode="wrap")
    x = ((x - x.min()) / (x.max() - x.min())).astype(np.float32) * np.float32(vr[1])
    x[0, 0, 3] = -1.0          # clipped to level 0
    x[0, H - 1, W - 2] = 9.0   # clipped to level M
    if batch == 1:
        src = ft.DeviceSource(torch.from_numpy(x[0]).cuda(), M, value_range=vr)
        got = [ft.descriptor_curves(src, _tabs(ft))]
        win = ft.descriptor_curves(ft.ArraySource(x[0], M, value_range=vr), _tabs(ft), chunk_bytes=3 * W * 4)
        assert all(np.array_equal(a.numerators, b.numerators) for a, b in zip(win, got[0]))
    else:
        got = ft.descriptor_curves_batch(torch.from_numpy(x).cuda(), M, _tabs(ft), value_range=vr)
    for b in range(batch):
        for c, w in zip(got[b], _want(orc, ft, x[b], M, vr)):
            assert np.array_equal(c.numerators, w), b


@pytest.mark.parametrize("H,batch", [(64, 1), (1, 1), (100, 3)])
def test_lines2d_stride_specialised_u8(ft, orc, H, batch):
    """W = 1024 u8 identity levels (the C3 kernels) on small stacks."""
    import torch
    rng = np.random.default_rng(H * 7 + batch)
    imgs = rng.integers(0, 256, size=(batch, H, 1024), dtype=np.uint8)
    got = ft.descriptor_curves_batch(imgs, 255, _tabs(ft)) if batch > 1 else \
        [ft.descriptor_curves(ft.DeviceSource(torch.from_numpy(imgs[0]).cuda(), 255), _tabs(ft))]
    for b in range(batch):
        for c, w in zip(got[b], _want(orc, ft, imgs[b], 255)):
            assert np.array_equal(c.numerators, w), b
