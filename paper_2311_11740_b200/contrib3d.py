"""3D vertex contributions (drop-in for fieldtopo.contrib3d, contrib3d.py:1-458).

``gather_3d_serial`` / ``gather_3d_parallel`` run the sm_100a kernel
``ft_hist3d`` (csrc/ft_hist3d.cu) and the device finalize; the returned
``ContributionMap3D`` is bit-identical to the reference's.  The per-vertex
helpers (``fill_data_3d``, ``accumulate_vertex_3d``) and the classifier
(``pair_classes``, ``classify_config``) are the reference's definitional
single-vertex API, kept for callers and tests.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import engine, gather
from ._tables import (SLOT_COORDS_3D, TYPE_NAMES_3D, ClassificationError, PairClassCounts,
                      classify_config, pair_classes)
from .sources import as_source

__all__ = ["ContributionMap3D", "VertexNeighborhood3D", "PairClassCounts", "ClassificationError",
           "fill_data_3d", "pair_classes", "classify_config", "accumulate_vertex_3d",
           "gather_3d_serial", "gather_3d_parallel", "TYPE_NAMES_3D", "SLOT_COORDS_3D"]


@dataclass(eq=False)
class ContributionMap3D:
    """Birth/death histograms per contribution type for one volume."""

    width: int
    height: int
    depth: int
    max_level: int
    q_in: np.ndarray   # (21, max_level + 2) uint64
    q_out: np.ndarray

    @classmethod
    def zeros(cls, width, height, depth, max_level):
        shape = (len(TYPE_NAMES_3D), max_level + 2)
        return cls(width, height, depth, max_level, np.zeros(shape, np.uint64), np.zeros(shape, np.uint64))

    ndim = property(lambda self: 3)
    type_names = property(lambda self: TYPE_NAMES_3D)

    @property
    def total_vertices(self):
        return (self.width + 1) * (self.height + 1) * (self.depth + 1)

    @property
    def cell_count(self):
        return self.width * self.height * self.depth

    def __eq__(self, other):
        return (isinstance(other, ContributionMap3D)
                and (self.width, self.height, self.depth, self.max_level)
                == (other.width, other.height, other.depth, other.max_level)
                and np.array_equal(self.q_in, other.q_in) and np.array_equal(self.q_out, other.q_out))

    def to_dict(self):
        return {"dimension": 3, "dims": {"w": self.width, "h": self.height, "d": self.depth},
                "max_level": self.max_level,
                "types": {n: {"in": self.q_in[t].tolist(), "out": self.q_out[t].tolist()}
                          for t, n in enumerate(TYPE_NAMES_3D)}}

    @classmethod
    def from_dict(cls, d):
        if d.get("dimension") != 3:
            raise ValueError("not a 3D contribution map")
        dims = d["dims"]
        m = cls.zeros(int(dims["w"]), int(dims["h"]), int(dims["d"]), int(d["max_level"]))
        for t, n in enumerate(TYPE_NAMES_3D):
            m.q_in[t] = np.asarray(d["types"][n]["in"], np.uint64)
            m.q_out[t] = np.asarray(d["types"][n]["out"], np.uint64)
        return m


@dataclass(frozen=True)
class VertexNeighborhood3D:
    """Levels of the eight cells around one vertex, in slot order."""

    data: tuple

    slot_coords = SLOT_COORDS_3D


def fill_data_3d(source, i, j, k):
    """Cell levels around vertex (i, j, k); absent cells take the sentinel
    (contrib3d.py:203-217)."""
    src = as_source(source)
    h, w, d, sent = src.height, src.width, src.depth, src.max_level + 1
    vals = []
    for ci, cj, ck in SLOT_COORDS_3D:
        p = (i - 1 + ci, j - 1 + cj, k - 1 + ck)
        inside = 0 <= p[0] < h and 0 <= p[1] < w and 0 <= p[2] < d
        vals.append(src.sample_at(*p) if inside else sent)
    return VertexNeighborhood3D(tuple(vals))


def accumulate_vertex_3d(nbhd, cmap):
    """Book one 3D neighbourhood: stage n (the n smallest levels, ties by
    slot) is born at sorted value n-1 and dies at sorted value n; stages >= 5
    are classified by their empty cells (contrib3d.py:220-238)."""
    data = nbhd.data
    order = sorted(range(8), key=lambda s: (data[s], s))
    for n in range(1, 9):
        group = order[:n] if n <= 4 else order[n:]
        t = classify_config(n, pair_classes(group))
        cmap.q_in[t, data[order[n - 1]]] += 1
        if n < 8:
            cmap.q_out[t, data[order[n]]] += 1
    return cmap


def _map_from_hist(src, hist):
    engine.check_classification(hist.device)  # contrib3d.py:425-426
    q_in, q_out, _ = engine.finalize(3, src.max_level, hist, maps=True)
    return ContributionMap3D(src.width, src.height, src.depth, src.max_level, engine.as_uint64(q_in),
                             engine.as_uint64(q_out))


def gather_3d_serial(source, device=None):
    """Contribution map of a volume over all (h+1)(w+1)(d+1) vertices, on the GPU."""
    src = as_source(source)
    return _map_from_hist(src, gather.source_hist(src, 3, device))


def gather_3d_parallel(source, workers, device=None, devices=None):
    """Same map as gather_3d_serial (see gather_2d_parallel for the knobs)."""
    src = as_source(source)
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if devices:
        return _map_from_hist(src, gather.multi_device_hist(src, 3, devices))
    return _map_from_hist(src, gather.source_hist(src, 3, device, workers=workers))
