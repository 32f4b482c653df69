"""The native runtime entry points of the C ABI (include/fieldtopo_b200.h):
ft_stream_begin / push / end (out-of-core streaming for non-Python callers;
reference _stream_rows_2d / _stream_slabs_3d, contrib2d.py:235-251,
contrib3d.py:392-414) and ft_multi_gather3d (slabs on several GPUs of one
process + one all-reduce; reference _parallel.py:8-33).  Every result is
compared bit for bit with the oracle (maps) or the reference curves."""
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


def _smooth(shape, seed):
    from scipy.ndimage import gaussian_filter
    x = gaussian_filter(np.random.default_rng(seed).standard_normal(shape).astype(np.float32), 1.7, mode="wrap")
    return ((x - x.min()) / (x.max() - x.min())).astype(np.float32)


def _maps(engine, ndim, M, hist):
    qi, qo, _ = engine.finalize(ndim, M, hist)
    return engine.as_uint64(qi), engine.as_uint64(qo)


@pytest.mark.parametrize("shape,chunk,push", [((23, 19, 31), 3, 1), ((23, 19, 31), 5, 7), ((40, 17, 64), 9, 40),
                                              ((5, 6, 7), 64, 2), ((61, 77), 4, 3), ((61, 77), 16, 61)])
def test_native_stream_maps_vs_oracle(ft, orc, shape, chunk, push):
    import torch
    from paper_2311_11740_b200 import engine
    x = _smooth(shape, len(shape) * 100 + chunk)
    M = 255
    q = ft.quant.QuantSpec.for_range(0.0, 1.0, M)
    g = orc.gather3d if len(shape) == 3 else orc.gather2d
    q_in, q_out = g(x, M, value_range=(0.0, 1.0), workers=8)
    for rows in (x, torch.from_numpy(x).pin_memory(), torch.from_numpy(x).cuda()):  # pageable, pinned, device
        hist = engine.stream_native(rows, shape, M, q, "map", chunk_rows=chunk, push_rows=push)
        qi, qo = _maps(engine, len(shape), M, hist)
        assert np.array_equal(qi, q_in) and np.array_equal(qo, q_out), type(rows)


@pytest.mark.parametrize("shape,chunk,push", [((33, 40, 70), 4, 5), ((33, 40, 70), 11, 33), ((50, 90), 6, 13)])
def test_native_stream_fused_curves(ft, orc, shape, chunk, push):
    from paper_2311_11740_b200 import engine, lattice
    x = _smooth(shape, 7)
    M = 511
    q = ft.quant.QuantSpec.for_range(0.0, 1.0, M)
    ndim = len(shape)
    if ndim == 3:
        tabs = [ft.builtin_weights(d, "26C") for d in ("ec", "surface-area", "volume")]
        q_in, q_out = orc.gather3d(x, M, value_range=(0.0, 1.0), workers=8)
    else:
        tabs = [ft.builtin_weights(*t) for t in (("ec", "8C"), ("perimeter", "8C"), ("area", "8C"))]
        q_in, q_out = orc.gather2d(x, M, value_range=(0.0, 1.0))
    plan = lattice.fused_plan(ndim, [t.eighths for t in tabs], lines_ok=ndim == 3)
    hist = engine.stream_native(x, shape, M, q, "fused", chunk_rows=chunk, push_rows=push)
    num = engine.curves_from_rows(hist, M, plan[2]).cpu().numpy() // plan[3][:, None]
    for c, t in zip(num, tabs):
        assert np.array_equal(c, orc.descriptor_numerators(q_in, q_out, M, t.eighths)), t.descriptor


def test_native_stream_argument_errors(ft):
    import ctypes

    from paper_2311_11740_b200 import _lib
    L = _lib.load()
    h = ctypes.c_void_p()
    q = _lib.ft_quant(0, 0, 0.0, 0.0, None)
    assert L.ft_stream_begin(4, 5, 5, 5, 0, ctypes.byref(q), 7, 0, 8, ctypes.c_void_p(1), None, ctypes.byref(h)) == 1
    assert L.ft_stream_begin(3, 5, 5, 5, 0, ctypes.byref(q), 7, 0, 2, ctypes.c_void_p(1), None, ctypes.byref(h)) == 1
    assert not h.value
    with pytest.raises(ValueError):  # ending before all rows arrived
        from paper_2311_11740_b200 import engine
        import torch
        hist = engine.new_hist(3, 7, torch.device("cuda", 0))
        assert L.ft_stream_begin(3, 5, 5, 5, 0, ctypes.byref(q), 7, 0, 3, ctypes.c_void_p(hist.data_ptr()), None,
                                 ctypes.byref(h)) == 0
        _lib.check(L.ft_stream_end(h), "ft_stream_end")


@pytest.mark.parametrize("kind", ["map", "fused"])
def test_multi_gather_slabs(ft, orc, kind):
    """Uneven slabs (split_blocks of H + 1 vertex rows), each holding only its
    own planes (+ the low halo); with one visible GPU the slabs share cuda:0
    (peer-copy reduction); on a multi-GPU box distinct devices take NCCL."""
    import torch

    from paper_2311_11740_b200 import engine, lattice
    from paper_2311_11740_b200._parallel import held_rows, split_blocks
    x = _smooth((37, 45, 66), 3)
    H, W, D = x.shape
    M = 255
    q = ft.quant.QuantSpec.for_range(0.0, 1.0, M)
    q_in, q_out = orc.gather3d(x, M, value_range=(0.0, 1.0), workers=8)
    tabs = [ft.builtin_weights(d, "26C") for d in ("ec", "surface-area", "volume")]
    plan = lattice.fused_plan(3, [t.eighths for t in tabs], lines_ok=True)
    ndev = torch.cuda.device_count()
    for nslab in (1, 2, 3, 5):
        parts = []
        for i, (a, b) in enumerate(split_blocks(H + 1, nslab)):
            r0, r1 = held_rows(a, b, H)
            parts.append((torch.from_numpy(x[r0:r1].copy()).to(f"cuda:{i % ndev}"), r0, (a, b)))
        hists, used_nccl = engine.multi_gather_native(parts, (H, W, D), M, q, kind)
        assert used_nccl == (ndev >= nslab > 1)
        for h in hists:
            if kind == "map":
                qi, qo = _maps(engine, 3, M, h)
                assert np.array_equal(qi, q_in) and np.array_equal(qo, q_out), nslab
            else:
                num = engine.curves_from_rows(h, M, plan[2]).cpu().numpy() // plan[3][:, None]
                for c, t in zip(num, tabs):
                    assert np.array_equal(c, orc.descriptor_numerators(q_in, q_out, M, t.eighths)), (nslab, t)
