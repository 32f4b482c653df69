"""GPU parity of the fused curve path (ft_lattice2d/3d, element histograms)
and the batched 2D API against the reference golden curves and the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

T2 = (("ec", "8C"), ("ec", "4C"), ("perimeter", "8C"), ("area", "8C"))
T3 = ("ec", "perimeter", "surface-area", "volume")


@pytest.fixture(scope="module")
def ft():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_11740_b200 as ft
    return ft


def test_lattice_2d_golden(ft, golden):
    tabs = [ft.builtin_weights(*t) for t in T2]
    for n in range(int(golden["n_f2d"])):
        lv, M = golden[f"f2d{n}_levels"], int(golden[f"f2d{n}_M"])
        curves = ft.descriptor_curves(ft.Field2D(lv, M), tabs, path="lattice")
        for t, c in enumerate(curves):
            assert np.array_equal(c.numerators, golden[f"f2d{n}_curves"][t]), (n, T2[t])


def test_lattice_3d_golden(ft, golden):
    tabs = [ft.builtin_weights(d, "26C") for d in ("ec", "surface-area", "volume")]
    for n in range(int(golden["n_f3d"])):
        lv, M = golden[f"f3d{n}_levels"], int(golden[f"f3d{n}_M"])
        curves = ft.descriptor_curves(ft.Field3D(lv, M), tabs, path="lattice")
        for c, t in zip(curves, (0, 2, 3)):
            assert np.array_equal(c.numerators, golden[f"f3d{n}_curves"][t]), (n, t)
    # the 3D sharp-edge perimeter is outside the lattice span: auto -> map path
    lv, M = golden["f3d9_levels"], int(golden["f3d9_M"])
    per = ft.descriptor_curves(ft.Field3D(lv, M), [ft.builtin_weights("perimeter", "26C")])[0]
    assert np.array_equal(per.numerators, golden["f3d9_curves"][1])
    with pytest.raises(ValueError):
        ft.descriptor_curves(ft.Field3D(lv, M), [ft.builtin_weights("perimeter", "26C")], path="lattice")


@pytest.mark.parametrize("shape,M,seed", [((1, 1, 1), 3, 0), ((1, 1, 7), 7, 1), ((9, 33, 1), 5, 2),
                                          ((17, 40, 65), 255, 3), ((33, 9, 31), 1, 4), ((8, 70, 130), 511, 5),
                                          ((5, 20, 64), 1023, 6), ((3, 70, 129), 2000, 7)])
def test_lattice_3d_vs_oracle(ft, orc, shape, M, seed):
    lv = np.random.default_rng(seed).integers(0, M + 1, size=shape, dtype=np.int32)
    q_in, q_out = orc.gather3d(lv, M, workers=8)
    tabs = [ft.builtin_weights(d, "26C") for d in ("ec", "surface-area", "volume")]
    for t, c in zip(tabs, ft.descriptor_curves(ft.Field3D(lv, M), tabs, path="lattice")):
        assert np.array_equal(c.numerators, orc.descriptor_numerators(q_in, q_out, M, t.eighths))


@pytest.mark.parametrize("dtype", [np.float32, np.uint16, np.uint8])
def test_lattice_3d_raw_dtypes(ft, orc, dtype):
    import torch
    rng = np.random.default_rng(9)
    if dtype == np.float32:
        x, vr, M = rng.random((24, 30, 38), dtype=np.float32), (0.0, 1.0), 511
    elif dtype == np.uint16:
        x, vr, M = rng.integers(0, 65536, (24, 30, 38)).astype(np.uint16), (0.0, 65535.0), 1023
    else:
        x, vr, M = rng.integers(0, 256, (24, 30, 37)).astype(np.uint8), None, 255
    q_in, q_out = orc.gather3d(x, M, value_range=vr, workers=8)
    src = ft.DeviceSource(torch.from_numpy(x).cuda(), M, value_range=vr)
    tabs = [ft.builtin_weights(d, "26C") for d in ("ec", "surface-area", "volume")]
    for t, c in zip(tabs, ft.descriptor_curves(src, tabs, path="lattice")):
        assert np.array_equal(c.numerators, orc.descriptor_numerators(q_in, q_out, M, t.eighths))


def test_lattice_2d_odd_and_float(ft, orc):
    import torch
    rng = np.random.default_rng(4)
    tabs = [ft.builtin_weights(*t) for t in T2]
    for shape in ((1, 1), (7, 1), (1, 9), (513, 1031), (64, 1024)):
        x = rng.random(shape, dtype=np.float32)
        q_in, q_out = orc.gather2d(x, 99, value_range=(0.0, 1.0), workers=8)
        src = ft.DeviceSource(torch.from_numpy(x).cuda(), 99, value_range=(0.0, 1.0))
        for t, c in zip(tabs, ft.descriptor_curves(src, tabs, path="lattice")):
            assert np.array_equal(c.numerators, orc.descriptor_numerators(q_in, q_out, 99, t.eighths)), shape


def test_lattice_streaming_equals_resident(ft, orc):
    rng = np.random.default_rng(12)
    x = rng.random((41, 30, 26), dtype=np.float32)
    q_in, q_out = orc.gather3d(x, 255, value_range=(0.0, 1.0), workers=8)
    tabs = [ft.builtin_weights(d, "26C") for d in ("ec", "surface-area", "volume")]
    want = [orc.descriptor_numerators(q_in, q_out, 255, t.eighths) for t in tabs]
    for chunk in (1, 5 * 30 * 26 * 4, 1 << 30):
        got = ft.descriptor_curves(ft.ArraySource(x, 255, value_range=(0.0, 1.0)), tabs, chunk_bytes=chunk)
        assert all(np.array_equal(c.numerators, w) for c, w in zip(got, want)), chunk
    import torch
    pinned = torch.from_numpy(x).pin_memory()
    got = ft.descriptor_curves(ft.ArraySource(pinned, 255, value_range=(0.0, 1.0)), tabs, chunk_bytes=4 * 30 * 26 * 4)
    assert all(np.array_equal(c.numerators, w) for c, w in zip(got, want))


def test_batch_2d_maps_and_curves(ft, orc):
    rng = np.random.default_rng(21)
    imgs = rng.integers(0, 256, size=(7, 33, 46), dtype=np.uint8)
    maps = ft.gather_2d_batch(imgs, 255)
    tabs = [ft.builtin_weights(*t) for t in T2]
    curves = ft.descriptor_curves_batch(imgs, 255, tabs)
    for b in range(imgs.shape[0]):
        q_in, q_out = orc.gather2d(imgs[b], 255)
        assert np.array_equal(maps[b].q_in, q_in) and np.array_equal(maps[b].q_out, q_out), b
        for t, c in zip(tabs, curves[b]):
            assert np.array_equal(c.numerators, orc.descriptor_numerators(q_in, q_out, 255, t.eighths)), b


def test_batch_2d_float_quantized(ft, orc):
    rng = np.random.default_rng(22)
    imgs = rng.random((5, 20, 31), dtype=np.float32)
    tabs = [ft.builtin_weights("ec", "8C")]
    curves = ft.descriptor_curves_batch(imgs, 63, tabs, value_range=(0.0, 1.0))
    for b in range(5):
        q_in, q_out = orc.gather2d(imgs[b], 63, value_range=(0.0, 1.0))
        assert np.array_equal(curves[b][0].numerators, orc.descriptor_numerators(q_in, q_out, 63, tabs[0].eighths))
