"""One process per GPU: z-slab (vertex-row) partition + one all-reduce.

The reference's only parallelism is contiguous vertex-row blocks on threads
with private histograms summed after the join (_parallel.py:8-33,
contrib2d.py:274-294, contrib3d.py:440-458).  Across GPUs the same contract
becomes:

* rank r owns vertex rows [v0, v1) = split_blocks(H + 1, world)[r] and holds
  cell planes [v0 - 2, v1 - 1] (its own planes plus the low halo planes:
  one for the vertex neighbourhoods, one for the per-cell signatures);
* each rank fills its histogram with the same kernels as a single GPU;
* one ``all_reduce(SUM)`` of the small histogram (NCCL over NVLink on GPUs,
  gloo on CPU) -- the only exchange step -- after which every rank holds the
  global histogram and finalizes the maps / curves itself.

Integer sums commute, so the result is bit-identical for any world size.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import engine, gather
from ._parallel import held_rows, split_blocks


@dataclass(frozen=True)
class Slab:
    """Rank-local part of a field of height H (rows 2D / planes 3D)."""

    rank: int
    world: int
    v0: int   # first vertex row owned
    v1: int   # one past the last vertex row owned
    r0: int   # first cell row/plane held (incl. the low halo)
    r1: int   # one past the last cell row/plane held

    @property
    def rows(self):
        return (self.v0, self.v1)

    @property
    def empty(self):
        return self.v1 <= self.v0


def slab_for(H, world, rank):
    """The slab of ``rank`` in a ``world``-way split of H + 1 vertex rows."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world size / rank")
    blocks = split_blocks(H + 1, world)
    if rank >= len(blocks):  # more ranks than vertex rows
        return Slab(rank, world, H + 1, H + 1, H, H)
    v0, v1 = blocks[rank]
    r0, r1 = held_rows(v0, v1, H)
    return Slab(rank, world, v0, v1, r0, r1)


def all_reduce_hist(hist, group=None):
    """Sum a histogram over the process group in place (the exchange step)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    return hist


def local_hist(ndim, x, shape, slab, M, quant, kind=gather.MAP):
    """This rank's histogram: ``x`` holds cell planes [slab.r0, slab.r1) of a
    field of global ``shape`` on this rank's GPU."""
    if slab.empty:
        return kind.new(ndim, M, x.device)
    return kind.launch(ndim, x, shape, M, quant, slab.rows, first=slab.r0)


def descriptor_curves_distributed(x, shape, max_level, tables, value_range=None, group=None):
    """Descriptor curves of a z-slab-partitioned field: every rank passes its
    planes [r0, r1) (``slab_for``) as a CUDA tensor and gets the global
    curves (identical on all ranks)."""
    import numpy as np
    import torch.distributed as dist

    from . import lattice
    from .descriptors import DescriptorCurve
    from .quant import QuantSpec

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    slab = slab_for(shape[0], world, rank)
    ndim = len(shape)
    M = int(max_level)
    quant = QuantSpec.for_range(*value_range, M) if value_range is not None else QuantSpec.identity()
    tables = list(tables)
    plan = None
    if engine.lattice_ok(ndim, shape, M):
        plan = lattice.fused_plan(ndim, [t.eighths for t in tables], lines_ok=ndim == 3 and engine.lines_ok(M))
    if plan is not None:
        hist = all_reduce_hist(local_hist(ndim, x, shape, slab, M, quant, gather.Kind(plan[0], plan[1])), group)
        num = engine.curves_from_rows(hist, M, plan[2]).cpu().numpy()
        num = num // plan[3][:, None]
    else:
        hist = all_reduce_hist(local_hist(ndim, x, shape, slab, M, quant), group)
        _, _, num = engine.finalize(ndim, M, hist, maps=False, tables=[t.eighths for t in tables])
        num = num.cpu().numpy()
    return [DescriptorCurve(t.descriptor, t.connectivity, M, num[i]) for i, t in enumerate(tables)]


def gather_distributed(x, shape, max_level, value_range=None, group=None):
    """Contribution map of a z-slab-partitioned field (every rank gets it)."""
    import torch.distributed as dist

    from .contrib2d import ContributionMap2D
    from .contrib3d import ContributionMap3D
    from .quant import QuantSpec

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    slab = slab_for(shape[0], world, rank)
    ndim = len(shape)
    M = int(max_level)
    quant = QuantSpec.for_range(*value_range, M) if value_range is not None else QuantSpec.identity()
    hist = all_reduce_hist(local_hist(ndim, x, shape, slab, M, quant), group)
    if ndim == 3:
        engine.check_classification(hist.device)
    q_in, q_out, _ = engine.finalize(ndim, M, hist, maps=True)
    qi, qo = engine.as_uint64(q_in), engine.as_uint64(q_out)
    if ndim == 2:
        return ContributionMap2D(shape[1], shape[0], M, qi, qo)
    return ContributionMap3D(shape[1], shape[0], shape[2], M, qi, qo)
