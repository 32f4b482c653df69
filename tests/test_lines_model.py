"""CPU model of the line-decomposition curve kernel (csrc/ft_lines.cu), pinned
to the reference golden curves (tests/golden, generated from the reference
itself), plus the host-side kernel choice.  No GPU needed.

The model books exactly what the kernel books: per cell a signature row
(u = #face neighbours first under the (level, index) order, s_i = the cell's
own A-line event) and, along every i-line of the min-derived families
B (j-1, j), C (k-1, k), D (both), +1 at a local minimum / -1 at a local
maximum (ties: lower i first).  EC_26C = A - B - C + D events, surface area =
2F - 6C, volume = C."""
import numpy as np
import pytest

EC, SA, VOL = 0, 2, 3  # golden curve order: ec, perimeter, surface-area, volume


def _hist(levels, M, w=None):
    h = np.zeros(M + 2, np.int64)
    np.add.at(h, levels.ravel(), 1 if w is None else w.ravel())
    return h


def _line_events(f, M):
    """chi of every i-line (axis 0) of levels f, by level: +1 local min, -1
    local max; sentinels M+1 beyond both ends; ties: lower i first."""
    S = M + 1
    g = np.concatenate([np.full((1,) + f.shape[1:], S), f, np.full((1,) + f.shape[1:], S)])
    c = g[1:-1]
    left_first = g[:-2] <= c
    right_first = g[2:] < c
    ev = (~left_first & ~right_first).astype(np.int64) - (left_first & right_first).astype(np.int64)
    return _hist(c, M, ev)


def lines_rows(levels, M):
    """(C, F, X = V - E) rows by level, as ft_lines3d accumulates them."""
    lv = np.asarray(levels, np.int64)
    H, W, D = lv.shape
    p = np.pad(lv, 1, constant_values=M + 1)
    q = p[1:H + 1]
    A = q[:, 1:W + 2, 1:D + 2]  # lattice positions (j, k) in [0, W] x [0, D]
    B = np.minimum(q[:, 0:W + 1, 1:D + 2], A)
    C = np.minimum(q[:, 1:W + 2, 0:D + 1], A)
    Dm = np.minimum(B, np.minimum(q[:, 0:W + 1, 0:D + 1], q[:, 1:W + 2, 0:D + 1]))
    ec = _line_events(A, M) - _line_events(B, M) - _line_events(C, M) + _line_events(Dm, M)
    # per-cell signature: faces whose other cell activates later are owned
    c = p[1:-1, 1:-1, 1:-1]
    u = np.zeros_like(c)
    for ax in range(3):
        lo = [slice(1, -1)] * 3
        hi = [slice(1, -1)] * 3
        lo[ax] = slice(0, -2)
        hi[ax] = slice(2, None)
        u += (p[tuple(lo)] <= c).astype(np.int64) + (p[tuple(hi)] < c).astype(np.int64)
    cells = _hist(c, M)
    faces = _hist(c, M, 6 - u)
    return cells, faces, ec - faces + cells


def curves(levels, M):
    cells, faces, x = lines_rows(levels, M)
    ec = np.cumsum(x + faces - cells)[:M + 1] * 8
    sa = np.cumsum(2 * faces - 6 * cells)[:M + 1] * 8
    vol = np.cumsum(cells)[:M + 1] * 8
    return ec, sa, vol


def test_model_matches_reference_golden_curves(golden):
    for n in range(int(golden["n_f3d"])):
        lv, M = golden[f"f3d{n}_levels"], int(golden[f"f3d{n}_M"])
        ec, sa, vol = curves(lv, M)
        want = golden[f"f3d{n}_curves"]
        assert np.array_equal(ec, want[EC]), n
        assert np.array_equal(sa, want[SA]), n
        assert np.array_equal(vol, want[VOL]), n


@pytest.mark.parametrize("seed", range(6))
def test_model_matches_oracle_random(orc, seed):
    rng = np.random.default_rng(100 + seed)
    shape = tuple(int(s) for s in rng.integers(1, 12, 3))
    M = int(rng.integers(0, 20))
    lv = rng.integers(0, M + 1, size=shape, dtype=np.int32)
    q_in, q_out = orc.gather3d(lv, M, workers=2)
    import paper_2311_11740_b200 as ft
    got = curves(lv, M)
    for t, g in zip(("ec", "surface-area", "volume"), got):
        want = orc.descriptor_numerators(q_in, q_out, M, ft.builtin_weights(t, "26C").eighths)
        assert np.array_equal(g, want), (seed, t)


def test_fused_plan_choice():
    import paper_2311_11740_b200 as ft
    from paper_2311_11740_b200 import lattice
    three = [ft.builtin_weights(d, "26C").eighths for d in ("ec", "surface-area", "volume")]
    plan = lattice.fused_plan(3, three)
    assert plan[0] == "lines" and plan[2].shape == (3, 3)
    # EC = X + F - C, surface area = 2F - 6C, volume = C (eighths)
    assert np.array_equal(plan[2] // plan[3][:, None], [[-8, 8, 8], [-48, 16, 0], [8, 0, 0]])
    assert lattice.fused_plan(3, three, lines_ok=False)[0] == "lattice"
    # the sharp-edge perimeter is in no fused span
    assert lattice.fused_plan(3, [ft.builtin_weights("perimeter", "26C").eighths]) is None
    assert lattice.fused_plan(2, [ft.builtin_weights("ec", "8C").eighths])[0] == "lattice"


def test_lines_level_limit():
    from paper_2311_11740_b200 import _lib
    L = _lib.load()
    assert L.ft_lines3d_ok(511) == 1 and L.ft_lines3d_ok(1023) == 1 and L.ft_lines3d_ok(2000) == 1
    assert L.ft_lines3d_ok(4000) == 0 and L.ft_lines3d_ok(-1) == 0


# ---- 2D (csrc/ft_lines2d.cu) -------------------------------------------------

def lines2d_rows(levels, M):
    """(C, E, V) rows by level as ft_lines2d accumulates them: signature rows
    (u = #edge neighbours first, s = the cell's own column-line event) and
    the events of the lines B_j = min over columns (j-1, j), j in [0, W];
    EC_8C = sum chi1(B) - sum chi1(A) (slicing along the lines between
    columns), V = EC + E - C."""
    lv = np.asarray(levels, np.int64)
    H, W = lv.shape
    p = np.pad(lv, 1, constant_values=M + 1)
    q = p[1:H + 1]
    A = q[:, 1:W + 2]  # lattice columns j in [0, W]
    B = np.minimum(q[:, 0:W + 1], A)
    ec = _line_events(B, M) - _line_events(A, M)
    c = p[1:-1, 1:-1]
    u = np.zeros_like(c)
    for ax in range(2):
        lo = [slice(1, -1)] * 2
        hi = [slice(1, -1)] * 2
        lo[ax] = slice(0, -2)
        hi[ax] = slice(2, None)
        u += (p[tuple(lo)] <= c).astype(np.int64) + (p[tuple(hi)] < c).astype(np.int64)
    cells = _hist(c, M)
    edges = _hist(c, M, 4 - u)
    return cells, edges, ec + edges - cells


def test_model2d_matches_reference_golden_curves(golden):
    for n in range(int(golden["n_f2d"])):
        lv, M = golden[f"f2d{n}_levels"], int(golden[f"f2d{n}_M"])
        cells, edges, verts = lines2d_rows(lv, M)
        want = golden[f"f2d{n}_curves"]  # ec 8C, ec 4C, perimeter, area
        assert np.array_equal(np.cumsum(verts - edges + cells)[:M + 1] * 8, want[0]), n
        assert np.array_equal(np.cumsum(2 * edges - 4 * cells)[:M + 1] * 8, want[2]), n
        assert np.array_equal(np.cumsum(cells)[:M + 1] * 8, want[3]), n


def test_lines2d_level_limit():
    from paper_2311_11740_b200 import _lib
    L = _lib.load()
    assert L.ft_lines2d_ok(255) == 1 and L.ft_lines2d_ok(1000) == 1
    assert L.ft_lines2d_ok(1100) == 0 and L.ft_lines2d_ok(-1) == 0
