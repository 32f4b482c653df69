"""Weight tables as integer combinations of the lattice histogram rows.

The fused curve kernels (``csrc/ft_lattice.cu``) count the elements of the
closed cubical complex by the level at which they appear:

* 3D rows: cells C, faces F, edges E, vertices V (min filters);
* 2D rows: cells C, edges E, vertices V (min filters), vertices V_max with
  every incident cell active (max filter).

Every vertex-type weight table of the reference (descriptors.py:27-48) that is
a linear combination of the tables "counting" those elements has the curve
``cumsum(sum_X r_X * H_X)`` with integer row weights r_X (eighths).  The
element-count tables follow from the reference builtins
(descriptors.py:83-97): C = volume / area, EC_26C = V - E + F - C,
surface area = 2F - 6C, EC_8C = V - E + C, EC_4C = -3C + E + V_max,
perimeter = 2E - 4C.  Tables outside the span (e.g. the 3D sharp-edge
"perimeter") use the transition-class map path instead.
"""

from __future__ import annotations

from fractions import Fraction
from functools import lru_cache

import numpy as np

# per-type eighths of one element count (type order TYPE_NAMES_2D/3D)
_C3 = np.array([1, 2, 2, 2, 3, 3, 3, 4, 4, 4, 4, 4, 4, 5, 5, 5, 6, 6, 6, 7, 8])
_EC3 = np.array([1, 0, -2, -6, -1, -3, -1, 0, -2, -2, 0, 0, 4, -1, 1, 3, 0, 2, 2, 1, 0])
_SA3 = np.array([6, 8, 12, 12, 10, 14, 18, 8, 12, 12, 16, 16, 24, 10, 14, 18, 8, 12, 12, 6, 0])
_V3 = np.full(21, 8)
_F3 = (_SA3 + 6 * _C3) // 2
_E3 = _V3 + _F3 - _C3 - _EC3
BASIS_3D = np.stack([_C3, _F3, _E3, _V3])          # rows: C, F, E, V
# rows of the line-decomposition kernel (ft_lines3d): C, F, X = V - E
BASIS_3D_LINES = np.stack([_C3, _F3, _V3 - _E3])

# E_max is not needed: per edge [min <= l] + [max <= l] = [a <= l] + [b <= l],
# so E + E_max = 4 C and EC_4C = C - E_max + V_max = -3 C + E + V_max.
BASIS_2D = np.array([[2, 4, 4, 6, 8],               # C
                     [8, 12, 16, 16, 16],           # E (any incident cell)
                     [8, 8, 8, 8, 8],               # V
                     [0, 0, 0, 0, 8]])              # V_max (all four cells)
_EMAX2 = np.array([0, 4, 0, 8, 16])
assert np.array_equal(BASIS_2D[1] + _EMAX2, 4 * BASIS_2D[0])
assert np.array_equal(BASIS_2D[2] - BASIS_2D[1] + BASIS_2D[0], [2, 0, -4, -2, 0])     # EC 8C
assert np.array_equal(BASIS_2D[0] - _EMAX2 + BASIS_2D[3], [2, 0, 4, -2, 0])          # EC 4C
assert np.array_equal(2 * BASIS_2D[1] - 4 * BASIS_2D[0], [8, 8, 16, 8, 0])          # perimeter
assert np.array_equal(BASIS_3D[3] - BASIS_3D[2] + BASIS_3D[1] - BASIS_3D[0], _EC3)


def _solve_exact(basis, w):
    """Rational coefficients c with c @ basis == w, or None."""
    B = [[Fraction(int(x)) for x in row] for row in basis]
    n, m = len(B), len(B[0])
    # Gaussian elimination on the transposed system basis^T c = w
    A = [[B[r][col] for r in range(n)] + [Fraction(int(w[col]))] for col in range(m)]
    piv_cols, row = [], 0
    for col in range(n):
        p = next((r for r in range(row, m) if A[r][col] != 0), None)
        if p is None:
            continue
        A[row], A[p] = A[p], A[row]
        A[row] = [x / A[row][col] for x in A[row]]
        for r in range(m):
            if r != row and A[r][col] != 0:
                f = A[r][col]
                A[r] = [a - f * b for a, b in zip(A[r], A[row])]
        piv_cols.append(col)
        row += 1
    if any(all(x == 0 for x in A[r][:n]) and A[r][n] != 0 for r in range(m)):
        return None
    c = [Fraction(0)] * n
    for r, col in enumerate(piv_cols):
        c[col] = A[r][n]
    return c


@lru_cache(maxsize=256)
def row_weights(ndim, eighths, rows="lattice"):
    """(integer row weights, divisor d) such that the table's curve
    numerators are cumsum(sum_X w_X H_X) / d; None if not expressible.
    ``rows``: "lattice" (ft_lattice2d/3d rows) or "lines" (ft_lines3d rows)."""
    if rows == "lines":
        basis = BASIS_3D_LINES if ndim == 3 else None
        if basis is None:
            return None
    else:
        basis = BASIS_3D if ndim == 3 else BASIS_2D
    c = _solve_exact(basis, eighths)
    if c is None:
        return None
    r = [8 * x for x in c]
    d = 1
    for x in r:
        d = d * x.denominator // np.gcd(d, x.denominator)
    return tuple(int(x * d) for x in r), d


def needs_max_rows(weights):
    """2D: whether the V_max row is used."""
    return len(weights) == 4 and weights[3] != 0


N_ROWS = {2: 4, 3: 4}


def fused_plan(ndim, tables_eighths, lines_ok=True):
    """Kernel choice for the fused curve path: ("lines" | "lattice", maxes,
    int64 row weights [n_tables, n_rows], divisors [n_tables]), or None when a
    table is outside the span of every fused kernel (the map path then)."""
    keys = [tuple(int(e) for e in t) for t in tables_eighths]
    if ndim == 3 and lines_ok:
        rw = [row_weights(3, k, "lines") for k in keys]
        if all(r is not None for r in rw):
            return "lines", False, np.array([r[0] for r in rw], np.int64), np.array([r[1] for r in rw], np.int64)
    rw = [row_weights(ndim, k) for k in keys]
    if any(r is None for r in rw):
        return None
    maxes = ndim == 2 and any(needs_max_rows(r[0]) for r in rw)
    return "lattice", maxes, np.array([r[0] for r in rw], np.int64), np.array([r[1] for r in rw], np.int64)
