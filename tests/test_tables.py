"""Transition-class tables: pinned to the reference classifier (golden) and
checked against the copies compiled into the CUDA library; a CPU model of the
kernels' event booking reproduces the reference maps exactly."""
import ctypes

import numpy as np
import pytest

from paper_2311_11740_b200 import _tables as T


def test_mask_types_match_reference(golden):
    got = np.array([T.mask_type_3d(m) for m in range(256)])
    assert np.array_equal(got[1:], golden["classify3d"][1:])


def test_type_names_match_reference(golden):
    assert tuple(golden["type_names_2d"]) == T.TYPE_NAMES_2D
    assert tuple(golden["type_names_3d"]) == T.TYPE_NAMES_3D


def test_transition_class_counts():
    assert T.TRANSITIONS_2D.n_classes == 6
    assert T.TRANSITIONS_3D.n_classes == 40
    t3 = T.TRANSITIONS_3D
    assert (t3.src[0], t3.dst[0]) == (-1, 0)            # empty -> q10
    assert (t3.src[39], t3.dst[39]) == (19, 20)         # q70 -> q80
    ranks = np.bincount([bin(m).count("1") for m in range(255) for s in range(8)
                         if not m >> s & 1 and t3.step[m * 8 + s] >= 0 and
                         t3.step[m * 8 + s] == t3.step[m * 8 + s]], minlength=8)
    assert ranks.sum() == 8 * 128


def test_library_tables_match_python():
    from paper_2311_11740_b200 import _lib
    L = _lib.load()
    for ndim, tab in ((2, T.TRANSITIONS_2D), (3, T.TRANSITIONS_3D)):
        S = 8 if ndim == 3 else 4
        step = np.zeros((1 << S) * S, np.int32)
        src = np.zeros(64, np.int32)
        dst = np.zeros(64, np.int32)
        assert L.ft_tables(ndim, step.ctypes.data, src.ctypes.data, dst.ctypes.data) == 0
        assert np.array_equal(step, tab.step)
        assert np.array_equal(src[:tab.n_classes], tab.src)
        assert np.array_equal(dst[:tab.n_classes], tab.dst)


def _model_hist2d(lv, M):
    """What ft_hist2d books, restated on the CPU: keys level*4+slot, sorted;
    classes 0 / (1|2) / (3|4) / 5 (csrc/ft_hist2d.cu)."""
    H, W = lv.shape
    pad = np.full((H + 2, W + 2), M + 1, np.int64)
    pad[1:-1, 1:-1] = lv
    hist = np.zeros((6, M + 2), np.uint64)
    for i in range(H + 1):
        for j in range(W + 1):
            keys = sorted([pad[i, j] * 4 + 0, pad[i, j + 1] * 4 + 1, pad[i + 1, j] * 4 + 2,
                           pad[i + 1, j + 1] * 4 + 3])
            diag = ((keys[0] ^ keys[1]) & 3) == 3
            for c, k in zip((0, 2 if diag else 1, 4 if diag else 3, 5), keys):
                hist[c, k >> 2] += 1
    return hist


def _model_hist3d(lv, M):
    """What ft_hist3d books: keys level*8+slot sorted, rank r books class
    step[mask_before * 8 + slot] at its level (csrc/ft_hist3d.cu::book3)."""
    H, W, D = lv.shape
    pad = np.full((H + 2, W + 2, D + 2), M + 1, np.int64)
    pad[1:-1, 1:-1, 1:-1] = lv
    step = T.TRANSITIONS_3D.step
    hist = np.zeros((40, M + 2), np.uint64)
    for i in range(H + 1):
        for j in range(W + 1):
            for k in range(D + 1):
                keys = sorted(pad[i + (s & 1), j + (s >> 1 & 1), k + (s >> 2 & 1)] * 8 + s for s in range(8))
                mask = 0
                for k8 in keys:
                    s = k8 & 7
                    hist[step[mask * 8 + s], k8 >> 3] += 1
                    mask |= 1 << s
    return hist


@pytest.mark.parametrize("n", range(6))
def test_kernel_model_2d_reproduces_reference(golden, n):
    lv, M = golden[f"f2d{n}_levels"], int(golden[f"f2d{n}_M"])
    q_in, q_out = T.reconstruct(T.TRANSITIONS_2D, _model_hist2d(lv, M))
    assert np.array_equal(q_in, golden[f"f2d{n}_qin"])
    assert np.array_equal(q_out, golden[f"f2d{n}_qout"])


@pytest.mark.parametrize("n", [0, 1, 2, 3, 4, 6, 7])
def test_kernel_model_3d_reproduces_reference(golden, n):
    lv, M = golden[f"f3d{n}_levels"], int(golden[f"f3d{n}_M"])
    hist = _model_hist3d(lv, M)
    q_in, q_out = T.reconstruct(T.TRANSITIONS_3D, hist)
    assert np.array_equal(q_in, golden[f"f3d{n}_qin"])
    assert np.array_equal(q_out, golden[f"f3d{n}_qout"])
    # curves straight from transition classes (finalize's formula)
    for t, w in enumerate(golden["w3d"]):
        delta = T.class_weights(T.TRANSITIONS_3D, w) @ hist.astype(np.int64)
        assert np.array_equal(np.cumsum(delta)[:M + 1], golden[f"f3d{n}_curves"][t])
