"""Configuration-type classification and the transition-class tables the
device kernels use.

Reference semantics restated here (host-side, table construction only):

* 2D types ``q1 q2 qd q3 q4`` (contrib2d.py:36); the two-face state is
  diagonal iff its two slots are NW+SE or NE+SW (contrib2d.py:134-136, 224).
* 3D types ``q10 .. q80`` (contrib3d.py:35-44), classified by the pair-class
  profile (n_face, n_edge, n_vertex) of the active cells for n <= 4 and of the
  empty cells for n >= 5 (contrib3d.py:76-135).

B200 design: every vertex neighbourhood walks stages
0 -> 1 -> ... -> 8 (3D) or 0 -> ... -> 4 (2D) as its sorted cell keys are
consumed.  Stage n dies exactly where stage n+1 is born, so instead of one
q_in and one q_out increment per stage the kernels book ONE event per sorted
rank into a histogram keyed by the *transition* (type_n -> type_{n+1}):
8 events per 3D vertex over 40 classes, 4 events per 2D vertex over 6
classes.  ``q_in``/``q_out`` and every descriptor curve are exact integer
sums of those histograms (``reconstruct`` below; ``finalize`` on device).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

TYPE_NAMES_2D = ("q1", "q2", "qd", "q3", "q4")
TYPE_NAMES_3D = (
    "q10",
    "q20", "q21", "q22",
    "q30", "q31", "q32",
    "q40", "q41", "q42", "q43", "q44", "q45",
    "q50", "q51", "q52",
    "q60", "q61", "q62",
    "q70",
    "q80",
)
_TYPE_INDEX_3D = {name: t for t, name in enumerate(TYPE_NAMES_3D)}

# Slot s of a 3D neighbourhood is the cell (i-1+di, j-1+dj, k-1+dk) with
# s = di + 2 dj + 4 dk (contrib3d.py:47-49).
SLOT_COORDS_3D = tuple((s & 1, (s >> 1) & 1, (s >> 2) & 1) for s in range(8))
# 2D slots [NW, NE, SW, SE] (contrib2d.py:39-40).
SLOT_COORDS_2D = ((0, 0), (0, 1), (1, 0), (1, 1))


class ClassificationError(RuntimeError):
    """A neighbourhood produced a pair-class profile outside the known table
    (contrib3d.py:54-55)."""


@dataclass(frozen=True)
class PairClassCounts:
    """Pairs at squared lattice distance 1 / 2 / 3 within a 2x2x2 block."""

    n_face: int
    n_edge: int
    n_vertex: int


def pair_classes(slots):
    """Pair-class counts for a set of slot indices (contrib3d.py:76-90)."""
    slots = list(slots)
    counts = [0, 0, 0]
    for a in range(len(slots)):
        for b in range(a + 1, len(slots)):
            counts[bin(slots[a] ^ slots[b]).count("1") - 1] += 1
    return PairClassCounts(*counts)


_PAIR = {(1, 0, 0): 0, (0, 1, 0): 1, (0, 0, 1): 2}
_TRIPLE = {(2, 1, 0): 0, (1, 1, 1): 1, (0, 3, 0): 2}
_QUAD = {(4, 2, 0): 0, (3, 3, 0): 1, (3, 2, 1): 2, (2, 3, 1): 3, (2, 2, 2): 4, (0, 6, 0): 5}
_STAGE_TABLE = {2: ("q20", _PAIR), 3: ("q30", _TRIPLE), 4: ("q40", _QUAD),
                5: ("q50", _TRIPLE), 6: ("q60", _PAIR)}


def classify_config(n, classes):
    """Type index for a configuration of n active cells (contrib3d.py:101-135).

    ``classes`` describes the active cells for n <= 4 and the empty cells for
    n >= 5; an unknown profile raises ClassificationError."""
    key = (classes.n_face, classes.n_edge, classes.n_vertex)
    if n in (1, 7, 8):
        if key == (0, 0, 0):
            return _TYPE_INDEX_3D[{1: "q10", 7: "q70", 8: "q80"}[n]]
    elif n in _STAGE_TABLE:
        base, table = _STAGE_TABLE[n]
        if key in table:
            return _TYPE_INDEX_3D[base] + table[key]
    raise ClassificationError(f"no configuration type for n={n}, classes={key}")


def mask_type_3d(mask):
    """Type of the stage whose active slots are ``mask`` (-1 for the empty
    stage)."""
    if mask == 0:
        return -1
    act = [s for s in range(8) if mask >> s & 1]
    emp = [s for s in range(8) if not mask >> s & 1]
    n = len(act)
    return classify_config(n, pair_classes(act if n <= 4 else emp))


def mask_type_2d(mask):
    n = bin(mask).count("1")
    if n == 0:
        return -1
    if n == 2:
        a, b = [s for s in range(4) if mask >> s & 1]
        return 2 if a + b == 3 else 1
    return {1: 0, 3: 3, 4: 4}[n]


@dataclass(frozen=True)
class TransitionTables:
    """Transition classes of one dimension.

    ``src[c]``/``dst[c]``: type that dies / is born at class c's event
    (-1 = the empty stage).  ``step[mask * S + slot]``: class booked when
    ``slot`` joins the active set ``mask`` (-1 where slot is already in mask).
    """

    ndim: int
    n_types: int
    src: np.ndarray
    dst: np.ndarray
    step: np.ndarray

    @property
    def n_classes(self):
        return len(self.src)


def _build(ndim):
    S = 8 if ndim == 3 else 4
    typ = mask_type_3d if ndim == 3 else mask_type_2d
    types = [typ(m) for m in range(1 << S)]
    pairs = set()
    for mask in range((1 << S) - 1):
        for s in range(S):
            if not mask >> s & 1:
                pairs.add((bin(mask).count("1"), types[mask], types[mask | 1 << s]))
    ordered = sorted(pairs)
    index = {(a, b): c for c, (_, a, b) in enumerate(ordered)}
    step = np.full((1 << S) * S, -1, np.int32)
    for mask in range((1 << S) - 1):
        for s in range(S):
            if not mask >> s & 1:
                step[mask * S + s] = index[(types[mask], types[mask | 1 << s])]
    src = np.array([a for _, a, _ in ordered], np.int32)
    dst = np.array([b for _, _, b in ordered], np.int32)
    n_types = len(TYPE_NAMES_3D) if ndim == 3 else len(TYPE_NAMES_2D)
    return TransitionTables(ndim, n_types, src, dst, step)


TRANSITIONS_2D = _build(2)
TRANSITIONS_3D = _build(3)
assert TRANSITIONS_2D.n_classes == 6 and TRANSITIONS_3D.n_classes == 40


def reconstruct(tables, hist):
    """Exact q_in / q_out (uint64 [T, M+2]) from a transition histogram
    [C, M+2] (host restatement of the device finalize, for tests)."""
    hist = np.asarray(hist, np.uint64)
    q_in = np.zeros((tables.n_types, hist.shape[-1]), np.uint64)
    q_out = np.zeros_like(q_in)
    for c in range(tables.n_classes):
        q_in[tables.dst[c]] += hist[c]
        if tables.src[c] >= 0:
            q_out[tables.src[c]] += hist[c]
    return q_in, q_out


def class_weights(tables, eighths):
    """Per-class curve delta (w_dst - w_src, eighths; w of the empty stage is 0)."""
    w = np.asarray(eighths, np.int64)
    return np.array([w[b] - (w[a] if a >= 0 else 0) for a, b in zip(tables.src, tables.dst)],
                    np.int64)
