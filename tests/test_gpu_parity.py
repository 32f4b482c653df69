"""GPU parity: the CUDA path (through the C ABI) against the reference golden
vectors and the CPU oracle, bit-exact (integer work: zero tolerance)."""
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


def _maps_equal(cmap, q_in, q_out):
    return np.array_equal(cmap.q_in, q_in) and np.array_equal(cmap.q_out, q_out)


def test_gather2d_golden(ft, golden):
    for n in range(int(golden["n_f2d"])):
        lv, M = golden[f"f2d{n}_levels"], int(golden[f"f2d{n}_M"])
        cmap = ft.gather_2d_serial(ft.Field2D(lv, M))
        assert _maps_equal(cmap, golden[f"f2d{n}_qin"], golden[f"f2d{n}_qout"]), n
        for t, name in enumerate([("ec", "8C"), ("ec", "4C"), ("perimeter", "8C"), ("area", "8C")]):
            c = ft.descriptor_curve(cmap, ft.builtin_weights(*name))
            assert np.array_equal(c.numerators, golden[f"f2d{n}_curves"][t]), (n, name)


def test_gather3d_golden(ft, golden):
    for n in range(int(golden["n_f3d"])):
        lv, M = golden[f"f3d{n}_levels"], int(golden[f"f3d{n}_M"])
        cmap = ft.gather_3d_serial(ft.Field3D(lv, M))
        assert _maps_equal(cmap, golden[f"f3d{n}_qin"], golden[f"f3d{n}_qout"]), n
        tabs = [ft.builtin_weights(d, "26C") for d in ("ec", "perimeter", "surface-area", "volume")]
        fused = ft.descriptor_curves(ft.Field3D(lv, M), tabs)
        for t, c in enumerate(fused):
            assert np.array_equal(c.numerators, golden[f"f3d{n}_curves"][t]), (n, t)


def test_config1_fused_quantize(ft, golden):
    import torch
    x = torch.from_numpy(golden["c1_x"]).cuda()
    src = ft.DeviceSource(x, 99, value_range=(0.0, 1.0))
    cmap = ft.gather_2d_serial(src)
    assert _maps_equal(cmap, golden["c1_qin"], golden["c1_qout"])
    tabs = [ft.builtin_weights(*t) for t in (("ec", "8C"), ("ec", "4C"), ("perimeter", "8C"), ("area", "8C"))]
    for t, c in enumerate(ft.descriptor_curves(src, tabs)):
        assert np.array_equal(c.numerators, golden["c1_curves"][t])


def test_config4_float_volume(ft, golden):
    import torch
    src = ft.DeviceSource(torch.from_numpy(golden["c4_x"]).cuda(), 255, value_range=(0.0, 1.0))
    assert _maps_equal(ft.gather_3d_serial(src), golden["c4_qin"], golden["c4_qout"])


def test_quantize_golden(ft, golden):
    for n in range(int(golden["n_quant"])):
        x = golden[f"quant{n}_x"]
        lo, hi, M = golden[f"quant{n}_params"]
        assert np.array_equal(ft.quantize_with_range(x, lo, hi, int(M)), golden[f"quant{n}_levels"]), n
        assert np.array_equal(ft.quantize_with_range(x.astype(np.float64), lo, hi, int(M)),
                              golden[f"quant{n}_levels"]), n
    assert np.array_equal(ft.quantize(golden["quant_u16_x"], 1023), golden["quant_u16_levels"])


@pytest.mark.parametrize("shape,M,seed", [((1, 1), 3, 0), ((1, 300), 7, 1), ((300, 1), 7, 2), ((257, 513), 255, 3),
                                          ((64, 1000), 1, 4), ((1025, 260), 63, 5)])
def test_gather2d_vs_oracle(ft, orc, shape, M, seed):
    lv = np.random.default_rng(seed).integers(0, M + 1, size=shape, dtype=np.int32)
    q_in, q_out = orc.gather2d(lv, M, workers=8)
    assert _maps_equal(ft.gather_2d_serial(ft.Field2D(lv, M)), q_in, q_out)


@pytest.mark.parametrize("shape,M,seed", [((1, 1, 1), 3, 0), ((1, 1, 70), 7, 1), ((9, 33, 1), 5, 2),
                                          ((17, 40, 65), 255, 3), ((33, 9, 31), 1, 4), ((8, 70, 100), 511, 5),
                                          ((5, 20, 64), 1023, 6)])
def test_gather3d_vs_oracle(ft, orc, shape, M, seed):
    lv = np.random.default_rng(seed).integers(0, M + 1, size=shape, dtype=np.int32)
    q_in, q_out = orc.gather3d(lv, M, workers=8)
    assert _maps_equal(ft.gather_3d_serial(ft.Field3D(lv, M)), q_in, q_out)


def test_smooth_float_field_3d_vs_oracle(ft, orc):
    import torch
    rng = np.random.default_rng(11)
    x = rng.standard_normal((40, 48, 56)).astype(np.float32)
    for ax in range(3):  # cheap smoothing: ties and long runs of near levels
        x = (x + np.roll(x, 1, ax) + np.roll(x, -1, ax)) / 3
    x = ((x - x.min()) / (x.max() - x.min())).astype(np.float32)
    q_in, q_out = orc.gather3d(x, 511, value_range=(0.0, 1.0), workers=8)
    cmap = ft.gather_3d_serial(ft.DeviceSource(torch.from_numpy(x).cuda(), 511, value_range=(0.0, 1.0)))
    assert _maps_equal(cmap, q_in, q_out)


def test_workers_and_devices_invariance(ft, golden):
    lv, M = golden["f3d9_levels"], int(golden["f3d9_M"])
    f = ft.Field3D(lv, M)
    ref = ft.gather_3d_serial(f)
    for w in (2, 3, 7, 64):
        assert ft.gather_3d_parallel(f, w) == ref
    assert ft.gather_3d_parallel(f, 1, devices=["cuda:0", "cuda:0"]) == ref
    with pytest.raises(ValueError):
        ft.gather_3d_parallel(f, 0)


def test_streaming_equals_resident(ft, orc):
    import paper_2311_11740_b200.gather as G
    rng = np.random.default_rng(5)
    x = rng.random((37, 29, 23), dtype=np.float32)
    src = ft.ArraySource(x, 63, value_range=(0.0, 1.0))
    q_in, q_out = orc.gather3d(x, 63, value_range=(0.0, 1.0), workers=8)
    for chunk in (1, 3 * 29 * 23 * 4, 10 * 29 * 23 * 4, 1 << 30):
        hist = G.stream_hist(src, 3, ft.engine.default_device(), (0, 38), chunk_bytes=chunk)
        from paper_2311_11740_b200 import engine
        qi, qo, _ = engine.finalize(3, 63, hist)
        assert np.array_equal(engine.as_uint64(qi), q_in) and np.array_equal(engine.as_uint64(qo), q_out), chunk


def test_lowmem_files(ft, golden, tmp_path):
    lv2 = golden["f2d9_levels"]
    f2 = ft.Field2D(lv2, 255)
    bmp = tmp_path / "a.bmp"
    ft.write_bmp(bmp, f2)
    with ft.open_bmp_lowmem(bmp) as src:
        assert ft.gather_2d_serial(src) == ft.gather_2d_serial(f2)
        assert src.peak_field_bytes > 0
    lv3 = golden["f3d9_levels"]
    f3 = ft.Field3D(lv3, 255)
    raw = tmp_path / "v.raw"
    ft.write_raw_volume(raw, f3, "u8")
    with ft.open_raw_lowmem(raw, (lv3.shape[1], lv3.shape[0], lv3.shape[2])) as src:
        assert ft.gather_3d_serial(src) == ft.gather_3d_serial(f3)


def test_u16_lowmem_auto_range(ft, orc, tmp_path):
    rng = np.random.default_rng(3)
    vol = rng.integers(100, 60000, size=(9, 10, 11)).astype(np.uint16)
    raw = tmp_path / "u16.raw"
    vol.tofile(raw)
    levels = orc.quantize(vol, 1023)
    ref = ft.gather_3d_serial(ft.Field3D(levels, 1023))
    with ft.open_raw_lowmem(raw, (10, 9, 11), "u16", 1023) as src:
        assert src.value_range == (float(vol.min()), float(vol.max()))
        assert ft.gather_3d_serial(src) == ref
    assert np.array_equal(ft.read_raw_volume(raw, (10, 9, 11), "u16", 1023).values, levels)


def test_counts_and_back_calc(ft, golden, orc):
    lv, M = golden["f2d6_levels"], int(golden["f2d6_M"])
    cmap = ft.gather_2d_serial(ft.Field2D(lv, M))
    counts = ft.counts_at_levels(cmap)
    assert np.array_equal(counts, orc.counts_at_levels(cmap.q_in, cmap.q_out, M))
    assert np.array_equal(ft.back_calc_empty(cmap), cmap.total_vertices - counts.sum(axis=0))


def test_random_field_normal_matches_reference_stream(ft, golden):
    # golden f3d4 = reference random_field((4, 3, 5), "normal", seed=7, max_level=6)
    f = ft.random_field((4, 3, 5), "normal", seed=7, max_level=6)
    assert np.array_equal(f.values, golden["f3d4_levels"])
