"""Raw-volume sources on the host side (no GPU): the reference's element
checks (sources.py:247-269, test_sources.py:243-247 -- float32 volumes are
rejected by read_raw_volume) and the streaming source's f32 addition."""
import numpy as np
import pytest

import paper_2311_11740_b200 as ft
from paper_2311_11740_b200.sources import RawVolumeSource


def _write(tmp_path, arr):
    p = tmp_path / "v.raw"
    arr.tofile(p)
    return p


def test_read_raw_volume_rejects_f32(tmp_path):
    p = _write(tmp_path, np.zeros((3, 4, 5), np.float32))
    with pytest.raises(ValueError):
        ft.read_raw_volume(p, (4, 3, 5), "f32", 255)


def test_stream_source_takes_f32_with_range(tmp_path):
    x = np.random.default_rng(0).random((3, 4, 5), dtype=np.float32)
    p = _write(tmp_path, x)
    with RawVolumeSource(p, (4, 3, 5), "f32", 511, value_range=(0.0, 1.0)) as src:
        assert src.shape == (3, 4, 5) and src.dtype == np.float32 and src.value_range == (0.0, 1.0)
        got = np.empty((2, 4, 5), np.float32)
        src.read_rows(1, 3, got)
        assert np.array_equal(got, x[1:3])


@pytest.mark.parametrize("element", ["f64", "u32", "i8"])
def test_stream_source_rejects_other_elements(tmp_path, element):
    p = _write(tmp_path, np.zeros(60, np.uint8))
    with pytest.raises(ValueError):
        RawVolumeSource(p, (4, 3, 5), element, 255, value_range=(0.0, 1.0))


def test_stream_source_size_mismatch(tmp_path):
    p = _write(tmp_path, np.zeros(59, np.float32))
    with pytest.raises(ValueError):
        RawVolumeSource(p, (4, 3, 5), "f32", 255, value_range=(0.0, 1.0))


def test_read_pencil_returns_decoded_levels_identity(tmp_path):
    # reference RawVolumeSource.read_pencil (sources.py:379-386) returns int32
    # levels, never the raw bytes
    vol = np.random.default_rng(1).integers(0, 256, size=(3, 4, 5)).astype(np.uint8)
    p = _write(tmp_path, vol)
    with ft.open_raw_lowmem(p, (4, 3, 5)) as src:
        pen = src.read_pencil(2, 1)
        assert pen.dtype == np.int32 and np.array_equal(pen, vol[2, 1].astype(np.int32))


def test_array_source_range_checks_identity_levels(tmp_path):
    # identity levels outside [0, M] raise like Field2D/3D (fields.py:48-59)
    ok = np.random.default_rng(2).integers(0, 8, size=(4, 5, 6)).astype(np.int32)
    ft.ArraySource(ok, 7)
    for bad in (ok + 1, ok - 1):
        with pytest.raises(ValueError, match=r"levels must lie in \[0, 7\]"):
            ft.ArraySource(bad, 7)
    with pytest.raises(ValueError):
        ft.ArraySource(np.full((3, 3), 9, np.uint8), 7)
    # memmaps are checked chunk by chunk as the engine stages them
    path = tmp_path / "m.i32"
    (ok + 1).tofile(path)
    mm = np.memmap(path, dtype=np.int32, mode="r", shape=ok.shape)
    src = ft.ArraySource(mm, 7)
    out = np.empty((2,) + ok.shape[1:], np.int32)
    with pytest.raises(ValueError):
        src.read_rows(0, 2, out)
    ft.ArraySource(np.full((3, 3), 2.5, np.float32), 7, value_range=(0.0, 8.0))  # samples: no check


BMP_DIR = __import__("pathlib").Path(__file__).resolve().parent / "golden" / "bmp"


@pytest.mark.parametrize("name", ["odd_7x5", "w8_8x3", "one_1x1"])
def test_bmp_matches_reference_writer_bytes(tmp_path, name):
    """write_bmp produces the reference writer's bytes (tests/golden/gen_bmp_golden.py)
    and read_bmp / BmpSource read them back top row first."""
    lv = np.load(BMP_DIR / f"{name}.npy")
    out = tmp_path / "x.bmp"
    ft.write_bmp(out, ft.Field2D(lv, 255))
    assert out.read_bytes() == (BMP_DIR / f"{name}.bmp").read_bytes()
    assert np.array_equal(ft.read_bmp(BMP_DIR / f"{name}.bmp").values, lv)
    with ft.open_bmp_lowmem(BMP_DIR / f"{name}.bmp") as src:
        assert (src.height, src.width) == lv.shape
        assert src.sample_at(lv.shape[0] - 1, 0) == lv[-1, 0]
        assert np.array_equal(src.read_row(0), lv[0].astype(np.uint8))
        got = np.empty(lv.shape, np.uint8)
        src.read_rows(0, lv.shape[0], got)
        assert np.array_equal(got, lv)


def test_bmp_top_down_and_errors(tmp_path):
    raw = bytearray((BMP_DIR / "odd_7x5.bmp").read_bytes())
    lv = np.load(BMP_DIR / "odd_7x5.npy")
    # negative stored height: rows stored top-down
    h = int.from_bytes(raw[22:26], "little", signed=True)
    off = int.from_bytes(raw[10:14], "little")
    stride = 8
    rows = [bytes(raw[off + r * stride: off + (r + 1) * stride]) for r in range(h)]
    td = raw[:off] + b"".join(rows[::-1])
    td[22:26] = (-h).to_bytes(4, "little", signed=True)
    p = tmp_path / "td.bmp"
    p.write_bytes(bytes(td))
    assert np.array_equal(ft.read_bmp(p).values, lv)
    cases = {"bad magic": b"XM" + bytes(raw[2:]), "truncated BMP file header": bytes(raw[:10]),
             "truncated BMP info header": bytes(raw[:30]), "truncated BMP pixel data": bytes(raw[:-3])}
    for msg, data in cases.items():
        p.write_bytes(data)
        with pytest.raises(ValueError, match=msg):
            ft.read_bmp(p)
    bad = bytearray(raw)
    bad[28:30] = (24).to_bytes(2, "little")
    p.write_bytes(bytes(bad))
    with pytest.raises(ValueError, match="only 8-bit BMP"):
        ft.read_bmp(p)
