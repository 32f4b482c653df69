"""GPU tests of API edges: single-image stacks in the batch API,
identity-level range checks on device sources, decoded read_pencil, and the
per-device guard of the library calls."""
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


@pytest.mark.parametrize("shape", [(1, 1), (1, 40), (37, 1), (23, 45)])
def test_batch_single_image_stack(ft, orc, shape):
    lv = np.random.default_rng(0).integers(0, 16, size=(1,) + shape, dtype=np.int32)
    q_in, q_out = orc.gather2d(lv[0], 15)
    (m,) = ft.gather_2d_batch(lv, 15)
    assert np.array_equal(m.q_in, q_in) and np.array_equal(m.q_out, q_out)
    tabs = [ft.builtin_weights("ec", "8C"), ft.builtin_weights("perimeter", "8C")]
    (cs,) = ft.descriptor_curves_batch(lv, 15, tabs)
    for c, t in zip(cs, tabs):
        assert np.array_equal(c.numerators, orc.descriptor_numerators(q_in, q_out, 15, t.eighths))


def test_device_source_rejects_out_of_range_levels(ft):
    import torch
    lv = torch.randint(0, 8, (5, 6, 7), dtype=torch.int32, device="cuda")
    ft.DeviceSource(lv, 7)
    for bad in (lv + 1, lv - 1):
        with pytest.raises(ValueError, match=r"levels must lie in \[0, 7\]"):
            ft.DeviceSource(bad, 7)
    with pytest.raises(ValueError):
        ft.DeviceSource(torch.full((4, 4), 200, dtype=torch.uint8, device="cuda"), 99)


def test_read_pencil_decodes_u16(ft, orc, tmp_path):
    vol = np.random.default_rng(3).integers(100, 60000, size=(4, 5, 6)).astype(np.uint16)
    p = tmp_path / "u16.raw"
    vol.tofile(p)
    levels = orc.quantize(vol, 1023)
    with ft.open_raw_lowmem(p, (5, 4, 6), "u16", 1023) as src:
        for i, j in ((0, 0), (3, 4), (2, 1)):
            pen = src.read_pencil(i, j)
            assert pen.dtype == np.int32 and np.array_equal(pen, levels[i, j])


def test_calls_follow_the_tensor_device(ft, orc):
    """Every library call runs with the tensor's device current (engine.on_device):
    a call made while another device context is active still lands on the
    tensor's device and stream (with one GPU visible: cuda:0 inside a
    cuda:0 context entered from elsewhere, plus the DeviceSource default)."""
    import torch
    from paper_2311_11740_b200 import engine
    x = np.random.default_rng(4).random((9, 10, 11), dtype=np.float32)
    q_in, q_out = orc.gather3d(x, 31, value_range=(0.0, 1.0))
    t = torch.from_numpy(x).cuda()
    src = ft.DeviceSource(t, 31, value_range=(0.0, 1.0))
    with engine.on_device(t.device):
        m = ft.gather_3d_serial(src)
    assert np.array_equal(m.q_in, q_in) and np.array_equal(m.q_out, q_out)
    if torch.cuda.device_count() > 1:  # a resident field is not moved to another GPU
        with pytest.raises(ValueError):
            ft.gather_3d_serial(src, device="cuda:1")


def test_read_bmp_device_decode(ft, orc, tmp_path):
    """BMP pixel decode (row flip + unpadding) on the device equals the host
    read_bmp (reference sources.py:154-164) on the reference writer's
    fixtures and on random sizes, and gathers like the host field."""
    from pathlib import Path
    bdir = Path(__file__).resolve().parent / "golden" / "bmp"
    for name in ("odd_7x5", "w8_8x3", "one_1x1"):
        src = ft.read_bmp_device(bdir / f"{name}.bmp")
        assert np.array_equal(src.tensor.cpu().numpy(), np.load(bdir / f"{name}.npy"))
    for shape in ((33, 61), (64, 64), (3, 130)):
        lv = np.random.default_rng(shape[1]).integers(0, 256, size=shape).astype(np.int32)
        p = tmp_path / "r.bmp"
        ft.write_bmp(p, ft.Field2D(lv, 255))
        src = ft.read_bmp_device(p)
        assert np.array_equal(src.tensor.cpu().numpy(), lv)
        q_in, q_out = orc.gather2d(lv, 255)
        m = ft.gather_2d_serial(src)
        assert np.array_equal(m.q_in, q_in) and np.array_equal(m.q_out, q_out)


def test_classification_trap_raises(ft, tmp_path, capsys):
    """A neighbourhood outside the configuration table raises
    ClassificationError (reference contrib3d.py:425-426) and the CLI exits
    with 2 (cli.py:271-273).  The real tables are total, so a corrupted table
    is installed for the test (ft_debug_trap_tables) and restored after."""
    from paper_2311_11740_b200 import _lib
    from paper_2311_11740_b200.cli import main
    L = _lib.load()
    f = ft.random_field((6, 5, 4), seed=1, max_level=15)
    good = ft.gather_3d_serial(f)
    _lib.check(L.ft_debug_trap_tables(1))
    try:
        with pytest.raises(ft.ClassificationError):
            ft.gather_3d_serial(f)
        assert main(["contrib-dump", "--generate", "6x5x4", "--seed", "1", "--max-level", "15"]) == 2
        assert "internal consistency" in capsys.readouterr().err
    finally:
        _lib.check(L.ft_debug_trap_tables(0))
    assert ft.gather_3d_serial(f) == good
