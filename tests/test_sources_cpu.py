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
