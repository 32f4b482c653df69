"""2D vertex contributions (drop-in for fieldtopo.contrib2d, contrib2d.py:1-294).

``gather_2d_serial`` / ``gather_2d_parallel`` run the sm_100a kernel
``ft_hist2d`` (csrc/ft_hist2d.cu) and the device finalize; the returned
``ContributionMap2D`` is bit-identical to the reference's.  The per-vertex
helpers (``neighborhood_data_2d``, ``diagonal_check``,
``accumulate_vertex_2d``) are the reference's definitional single-vertex API,
kept for callers and tests; they never run inside a gather.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import engine, gather
from ._tables import SLOT_COORDS_2D, TYPE_NAMES_2D
from .sources import as_source

Q1, Q2, QD, Q3, Q4 = range(5)


@dataclass(eq=False)
class ContributionMap2D:
    """Birth/death histograms per contribution type for one 2D field."""

    width: int
    height: int
    max_level: int
    q_in: np.ndarray   # (5, max_level + 2) uint64
    q_out: np.ndarray

    @classmethod
    def zeros(cls, width, height, max_level):
        shape = (len(TYPE_NAMES_2D), max_level + 2)
        return cls(width, height, max_level, np.zeros(shape, np.uint64), np.zeros(shape, np.uint64))

    ndim = property(lambda self: 2)
    type_names = property(lambda self: TYPE_NAMES_2D)

    @property
    def total_vertices(self):
        return (self.width + 1) * (self.height + 1)

    @property
    def cell_count(self):
        return self.width * self.height

    def __eq__(self, other):
        return (isinstance(other, ContributionMap2D)
                and (self.width, self.height, self.max_level) == (other.width, other.height, other.max_level)
                and np.array_equal(self.q_in, other.q_in) and np.array_equal(self.q_out, other.q_out))

    def to_dict(self):
        return {"dimension": 2, "dims": {"w": self.width, "h": self.height}, "max_level": self.max_level,
                "types": {n: {"in": self.q_in[t].tolist(), "out": self.q_out[t].tolist()}
                          for t, n in enumerate(TYPE_NAMES_2D)}}

    @classmethod
    def from_dict(cls, d):
        if d.get("dimension") != 2:
            raise ValueError("not a 2D contribution map")
        m = cls.zeros(int(d["dims"]["w"]), int(d["dims"]["h"]), int(d["max_level"]))
        for t, n in enumerate(TYPE_NAMES_2D):
            m.q_in[t] = np.asarray(d["types"][n]["in"], np.uint64)
            m.q_out[t] = np.asarray(d["types"][n]["out"], np.uint64)
        return m


@dataclass(frozen=True)
class VertexNeighborhood2D:
    """Levels of the four faces around one vertex, ordered [NW, NE, SW, SE]."""

    data: tuple

    slot_coords = SLOT_COORDS_2D


def neighborhood_data_2d(source, i, j):
    """Face levels around vertex (i, j) with independent bounds checks;
    absent faces take the sentinel max_level + 1 (contrib2d.py:117-131)."""
    src = as_source(source)
    h, w, sent = src.height, src.width, src.max_level + 1
    vals = []
    for di, dj in SLOT_COORDS_2D:
        r, c = i - 1 + di, j - 1 + dj
        vals.append(src.sample_at(r, c) if 0 <= r < h and 0 <= c < w else sent)
    return VertexNeighborhood2D(tuple(vals))


def diagonal_check(pos0, pos1):
    """True when two distinct 2x2 slots touch only at the centre."""
    return pos0[0] != pos1[0] and pos0[1] != pos1[1]


def accumulate_vertex_2d(nbhd, cmap):
    """Book one neighbourhood (stable sort by slot on ties; contrib2d.py:139-158)."""
    data = nbhd.data
    order = sorted(range(4), key=lambda s: (data[s], s))
    v = [data[s] for s in order]
    two = QD if diagonal_check(SLOT_COORDS_2D[order[0]], SLOT_COORDS_2D[order[1]]) else Q2
    for t, born, dies in ((Q1, v[0], v[1]), (two, v[1], v[2]), (Q3, v[2], v[3]), (Q4, v[3], None)):
        cmap.q_in[t, born] += 1
        if dies is not None:
            cmap.q_out[t, dies] += 1
    return cmap


def _map_from_hist(src, hist):
    q_in, q_out, _ = engine.finalize(2, src.max_level, hist, maps=True)
    return ContributionMap2D(src.width, src.height, src.max_level, engine.as_uint64(q_in),
                             engine.as_uint64(q_out))


def gather_2d_serial(source, device=None):
    """Contribution map of a 2D field over all (h+1)(w+1) vertices, on the GPU."""
    src = as_source(source)
    return _map_from_hist(src, gather.source_hist(src, 2, device))


def gather_2d_parallel(source, workers, device=None, devices=None):
    """Same map as gather_2d_serial.  ``workers`` keeps the reference's row-block
    contract (ValueError below 1; one launch per block); ``devices`` spreads
    vertex-row slabs over several GPUs of this process."""
    src = as_source(source)
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if devices:
        return _map_from_hist(src, gather.multi_device_hist(src, 2, devices))
    return _map_from_hist(src, gather.source_hist(src, 2, device, workers=workers))
