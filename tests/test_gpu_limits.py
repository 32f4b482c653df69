"""GPU parity on BOTH sides of every level-count switch point of the
kernels (bit-exact against the pinned oracle): the 3D map kernel's
lane-replicated rank tables (M <= 601) vs the 4096-entry ones, the 2D map
kernel's byte-offset keys (M <= 2728) vs word indices, the line kernels'
folded signature rows (3D, M <= 763) and their 16-bit bin offsets (the last
M ft_lines3d / ft_lines2d take, then the lattice kernels)."""
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


def _levels(shape, M, seed):
    """Uniform levels with the extremes 0 and M forced in (first / last bins)."""
    lv = np.random.default_rng(seed).integers(0, M + 1, size=shape, dtype=np.int32)
    lv.flat[0], lv.flat[-1] = 0, M
    return lv


@pytest.mark.parametrize("M", [599, 600, 601, 602, 603, 700])
def test_map3d_rank_table_switch(ft, orc, M):
    lv = _levels((5, 70, 131), M, M)
    m = ft.gather_3d_serial(ft.Field3D(lv, M))
    q_in, q_out = orc.gather3d(lv, M, workers=8)
    assert np.array_equal(m.q_in, q_in) and np.array_equal(m.q_out, q_out)


@pytest.mark.parametrize("M", [2264, 2265, 2266, 2727, 2728, 2729, 2730, 3000])
def test_map2d_key_form_switch(ft, orc, M):
    lv = _levels((37, 200), M, M)
    m = ft.gather_2d_serial(ft.Field2D(lv, M))
    q_in, q_out = orc.gather2d(lv, M, workers=4)
    assert np.array_equal(m.q_in, q_in) and np.array_equal(m.q_out, q_out)


def _last_ok(ok, lo, hi):
    assert ok(lo) and not ok(hi)
    while hi - lo > 1:
        mid = (lo + hi) // 2
        lo, hi = (mid, hi) if ok(mid) else (lo, mid)
    return lo


def _curves3d(ft, orc, lv, M, path):
    tabs = [ft.builtin_weights(d, "26C") for d in ("ec", "surface-area", "volume")]
    q_in, q_out = orc.gather3d(lv, M, workers=8)
    got = ft.descriptor_curves(ft.Field3D(lv, M), tabs, path=path)
    for c, t in zip(got, tabs):
        assert np.array_equal(c.numerators, orc.descriptor_numerators(q_in, q_out, M, t.eighths)), (M, path, t.descriptor)


@pytest.mark.parametrize("M", [762, 763, 764, 765, 766, 1023])
def test_lines3d_fold_switch(ft, orc, M):
    """21 folded signature rows up to M = 763, then 7 rows + A-line events."""
    _curves3d(ft, orc, _levels((6, 40, 131), M, M), M, "lines")


def test_lines3d_last_level_count(ft, orc):
    from paper_2311_11740_b200 import engine
    last = _last_ok(engine.lines_ok, 1023, 5000)
    assert 2000 < last < 2400  # 7 rows of (M + 2) * 4 bytes in 16-bit offsets
    for M in (last - 1, last):
        _curves3d(ft, orc, _levels((4, 20, 70), M, M), M, "lines")
    lv = _levels((4, 20, 70), last + 1, 5)
    with pytest.raises(ValueError):
        ft.descriptor_curves(ft.Field3D(lv, last + 1), [ft.builtin_weights("ec", "26C")], path="lines")
    _curves3d(ft, orc, lv, last + 1, "auto")  # served by the lattice kernel


def test_lines2d_last_level_count(ft, orc):
    from paper_2311_11740_b200 import engine
    last = _last_ok(engine.lines2d_ok, 255, 5000)
    assert 900 < last < 1200  # 15 signature rows in 16-bit offsets
    tabs = [ft.builtin_weights(d, "8C") for d in ("ec", "perimeter", "area")]
    for M in (last - 1, last, last + 1, last + 2):  # the last two: lattice kernel
        lv = _levels((40, 200), M, M)
        q_in, q_out = orc.gather2d(lv, M, workers=4)
        got = ft.descriptor_curves(ft.Field2D(lv, M), tabs)
        for c, t in zip(got, tabs):
            assert np.array_equal(c.numerators, orc.descriptor_numerators(q_in, q_out, M, t.eighths)), (M, t.descriptor)
