"""Row-block partitioning with the reference's block contract
(_parallel.py:8-24: equal blocks of total // workers, the remainder on the
last block, empty blocks dropped).

On the GPU the same contiguous vertex-row blocks become launch ranges,
per-GPU slabs (``gather.multi_device_hist``) and per-rank slabs
(``distributed``); every partition gives the identical histogram.
"""

from __future__ import annotations


def split_blocks(total, workers):
    if workers < 1:
        raise ValueError("workers must be >= 1")
    step = total // workers
    edges = [w * step for w in range(workers)] + [total]
    return [(lo, hi) for lo, hi in zip(edges[:-1], edges[1:]) if hi > lo]
