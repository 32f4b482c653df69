"""GPU parity of the line-decomposition curve kernel (ft_lines3d) -- the
default fused path for 3D EC / surface-area / volume -- against the reference
golden curves and the pinned oracle, bit-exact.  Shapes cover boundary-only
tiles, interior warp strips (guard-free loop), several plane chunks, the
FOLD (M <= ~770) and unfolded signature layouts, every quantizer."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
T3 = ("ec", "surface-area", "volume")


@pytest.fixture(scope="module")
def ft():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_11740_b200 as ft
    return ft


def _tabs(ft):
    return [ft.builtin_weights(d, "26C") for d in T3]


def _want(orc, ft, x, M, vr=None):
    q_in, q_out = orc.gather3d(x, M, value_range=vr, workers=16)
    return [orc.descriptor_numerators(q_in, q_out, M, t.eighths) for t in _tabs(ft)]


def test_lines_golden(ft, golden):
    for n in range(int(golden["n_f3d"])):
        lv, M = golden[f"f3d{n}_levels"], int(golden[f"f3d{n}_M"])
        curves = ft.descriptor_curves(ft.Field3D(lv, M), _tabs(ft), path="lines")
        for c, t in zip(curves, (0, 2, 3)):
            assert np.array_equal(c.numerators, golden[f"f3d{n}_curves"][t]), (n, t)


@pytest.mark.parametrize("shape,M,seed", [((1, 1, 1), 3, 0), ((1, 1, 7), 7, 1), ((9, 33, 1), 5, 2),
                                          ((17, 40, 65), 255, 3), ((33, 9, 31), 1, 4), ((8, 70, 130), 511, 5),
                                          ((5, 20, 64), 1023, 6), ((3, 70, 129), 2000, 7),
                                          ((140, 45, 190), 0, 8), ((150, 41, 187), 2, 9)])
def test_lines_vs_oracle_levels(ft, orc, shape, M, seed):
    lv = np.random.default_rng(seed).integers(0, M + 1, size=shape, dtype=np.int32)
    got = ft.descriptor_curves(ft.Field3D(lv, M), _tabs(ft), path="lines")
    for c, w in zip(got, _want(orc, ft, lv, M)):
        assert np.array_equal(c.numerators, w)


def _grf(shape, sigma, seed):
    from scipy.ndimage import gaussian_filter
    x = gaussian_filter(np.random.default_rng(seed).standard_normal(shape).astype(np.float32), sigma, mode="wrap")
    return ((x - x.min()) / (x.max() - x.min())).astype(np.float32)


@pytest.mark.parametrize("vr,M", [((0.0, 1.0), 511), ((0.0, 1.0), 255), ((0.05, 0.95), 511), ((0.0, 2.0), 1023)])
def test_lines_interior_float(ft, orc, vr, M):
    """Smooth f32 fields big enough for interior strips and 3 plane chunks:
    the guard-free loop, FMUL.SAT quantizer (pow2 ranges) and table path."""
    import torch
    x = _grf((200, 90, 260), 3.0, 31 + M)
    x[100, 50, 130] = -3.0  # out-of-range cells quantize like the reference (level 0 / M)
    x[150, 60, 140] = 7.0
    src = ft.DeviceSource(torch.from_numpy(x).cuda(), M, value_range=vr)
    got = ft.descriptor_curves(src, _tabs(ft), path="lines")
    for c, w in zip(got, _want(orc, ft, x, M, vr)):
        assert np.array_equal(c.numerators, w)


@pytest.mark.parametrize("dtype", [np.uint16, np.uint8])
def test_lines_interior_int(ft, orc, dtype):
    import torch
    x = _grf((180, 75, 200), 2.5, 7)
    if dtype == np.uint16:
        raw, vr, M = np.floor(x * 65535 + 0.5).astype(np.uint16), (0.0, 65535.0), 1023
    else:
        raw, vr, M = np.floor(x * 255 + 0.5).astype(np.uint8), None, 255
    src = ft.DeviceSource(torch.from_numpy(raw).cuda(), M, value_range=vr)
    got = ft.descriptor_curves(src, _tabs(ft), path="lines")
    for c, w in zip(got, _want(orc, ft, raw, M, vr)):
        assert np.array_equal(c.numerators, w)


def test_lines_slabs_and_streaming(ft, orc):
    """Row blocks (workers=) and pinned chunk streaming give the same curves."""
    import torch
    x = _grf((170, 64, 128), 2.0, 77)
    want = _want(orc, ft, x, 511, (0.0, 1.0))
    src = ft.DeviceSource(torch.from_numpy(x).cuda(), 511, value_range=(0.0, 1.0))
    for workers in (1, 2, 5):
        got = ft.descriptor_curves(src, _tabs(ft), workers=workers, path="lines")
        assert all(np.array_equal(c.numerators, w) for c, w in zip(got, want)), workers
    for chunk in (3 * 64 * 128 * 4, 40 * 64 * 128 * 4, 1 << 30):
        got = ft.descriptor_curves(ft.ArraySource(x, 511, value_range=(0.0, 1.0)), _tabs(ft), chunk_bytes=chunk)
        assert all(np.array_equal(c.numerators, w) for c, w in zip(got, want)), chunk


def test_lines_auto_and_limits(ft, orc):
    lv = np.random.default_rng(3).integers(0, 3001, size=(6, 7, 8), dtype=np.int32)
    with pytest.raises(ValueError):  # M = 3000 exceeds ft_lines3d's 16-bit row offsets
        ft.descriptor_curves(ft.Field3D(lv, 3000), _tabs(ft), path="lines")
    got = ft.descriptor_curves(ft.Field3D(lv, 3000), _tabs(ft))  # auto -> lattice kernel
    for c, w in zip(got, _want(orc, ft, lv, 3000)):
        assert np.array_equal(c.numerators, w)


@pytest.mark.parametrize("D", [61, 62, 63, 64, 123, 124, 125, 126, 127, 186, 187, 188, 189, 256, 512])
def test_lines_column_tiles(ft, orc, D):
    """Row lengths around the 62-column warp-strip tiling (interior / k-boundary
    tile split, the halo halves of lanes 0 and 31) and the D-specialised
    interior loads (256, 512), on a smooth f32 field with the pow2 quantizer."""
    import torch
    x = _grf((37, 70, D), 2.0, 1000 + D)
    src = ft.DeviceSource(torch.from_numpy(x).cuda(), 511, value_range=(0.0, 1.0))
    got = ft.descriptor_curves(src, _tabs(ft), path="lines")
    for c, w in zip(got, _want(orc, ft, x, 511, (0.0, 1.0))):
        assert np.array_equal(c.numerators, w)


def test_lines_streaming_short_segments(ft, orc):
    """Pinned streaming in windows of a few planes over a field wide enough
    that the even CTA split cuts the windows into segments of one or two
    planes: the march must not read past a window's last plane."""
    import torch
    x = _grf((23, 200, 190), 2.0, 91)
    want = _want(orc, ft, x, 511, (0.0, 1.0))
    for planes in (3, 4, 7):
        got = ft.descriptor_curves(ft.ArraySource(x, 511, value_range=(0.0, 1.0)), _tabs(ft),
                                   chunk_bytes=planes * 200 * 190 * 4)
        assert all(np.array_equal(c.numerators, w) for c, w in zip(got, want)), planes


def test_lines_raw_f32_streaming(ft, orc, tmp_path):
    """Headerless float32 volume streamed from the file (RawVolumeSource
    element "f32", the out-of-core entry point of SURVEY.md §8f row 3), with
    an explicit range and with the streaming device min/max pass."""
    from paper_2311_11740_b200.sources import RawVolumeSource
    x = _grf((41, 70, 130), 2.0, 55)
    x = (x * 3.0 - 1.0).astype(np.float32)  # range [-1, 2]: not a power-of-two span
    p = tmp_path / "f.raw"
    x.tofile(p)
    for vr in ((-1.0, 2.0), None):
        with RawVolumeSource(p, (70, 41, 130), "f32", 511, value_range=vr, chunk_bytes=1 << 20) as src:
            want = _want(orc, ft, x, 511, src.value_range)
            if vr is None:
                assert src.value_range == (float(x.min()), float(x.max()))
            got = ft.descriptor_curves(src, _tabs(ft), chunk_bytes=7 * 70 * 130 * 4)
            assert all(np.array_equal(c.numerators, w) for c, w in zip(got, want)), vr


@pytest.mark.parametrize("dtype,D,vr,M", [(np.float32, 1024, (0.0, 1.0), 511), (np.float32, 2048, (0.0, 1.0), 511),
                                          (np.float32, 1024, (0.1, 0.9), 255), (np.float32, 2048, (0.0, 2.0), 1023),
                                          (np.uint16, 512, (0.0, 65535.0), 1023), (np.uint16, 1024, (0.0, 65535.0), 255),
                                          (np.uint16, 2048, (0.0, 65535.0), 511)])
def test_lines_row_length_specialised(ft, orc, dtype, D, vr, M):
    """The D-specialised instantiations (immediate-offset row loads; 256 /
    512 / 1024 / 2048 for f32 pow2 + table and u16 table inputs) on fields
    small enough for the oracle, incl. the k-boundary tiles of those lengths."""
    import torch
    x = _grf((11, 70, D), 2.0, D + M)
    if dtype == np.uint16:
        x = np.floor(x * 65535 + 0.5).astype(np.uint16)
    else:
        x = x * np.float32(vr[1])
        x[3, 5, D - 1] = -1.0   # clipped to level 0
        x[7, 69, 0] = 10.0      # clipped to level M
    src = ft.DeviceSource(torch.from_numpy(x).cuda(), M, value_range=vr)
    got = ft.descriptor_curves(src, _tabs(ft), path="lines")
    for c, w in zip(got, _want(orc, ft, x, M, vr)):
        assert np.array_equal(c.numerators, w)
