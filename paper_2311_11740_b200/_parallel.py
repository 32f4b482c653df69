"""Row-block partitioning with the reference's block contract
(_parallel.py:8-24: equal blocks of total // workers, the remainder on the
last block, empty blocks dropped).

On the GPU the same contiguous vertex-row blocks become launch ranges,
per-GPU slabs (``gather.multi_device_hist``) and per-rank slabs
(``distributed``); every partition gives the identical histogram.
"""

from __future__ import annotations

# Cell rows/planes below its first vertex row a slab must hold: vertex row a
# reads planes a-1 and a; the fused-curve kernel also signs the cells of
# plane a-1, whose -i neighbour is plane a-2.
LOW_HALO = 2


def held_rows(v0, v1, H):
    """Cell rows/planes [r0, r1) a slab of vertex rows [v0, v1) holds."""
    r0 = max(v0 - LOW_HALO, 0)
    r1 = max(min(v1 - 1, H - 1) + 1, r0)
    return r0, r1


def split_blocks(total, workers):
    if workers < 1:
        raise ValueError("workers must be >= 1")
    step = total // workers
    edges = [w * step for w in range(workers)] + [total]
    return [(lo, hi) for lo, hi in zip(edges[:-1], edges[1:]) if hi > lo]
