"""Multi-rank host logic on CPU (gloo, world_size 2): z-slab plans and the
histogram all-reduce give the single-process result bit for bit.  The
per-rank histograms here come from the CPU oracle (test infrastructure); on
GPUs the same driver fills them with the CUDA kernels and NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2311_11740_b200._parallel import split_blocks
from paper_2311_11740_b200.distributed import all_reduce_hist, slab_for


def test_slab_plan_covers_every_vertex_row():
    for H in (1, 2, 7, 100, 2048):
        for world in (1, 2, 3, 4, 8, 16):
            slabs = [slab_for(H, world, r) for r in range(world)]
            rows = [v for s in slabs for v in range(s.v0, s.v1)]
            assert rows == list(range(H + 1))
            for s in slabs:
                if not s.empty:  # planes needed by vertex rows [v0, v1) (+ the signature halo)
                    assert s.r0 == max(s.v0 - 2, 0) and s.r1 == min(s.v1 - 1, H - 1) + 1
    assert [(s.v0, s.v1) for s in (slab_for(10, 3, r) for r in range(3))] == split_blocks(11, 3)
    with pytest.raises(ValueError):
        slab_for(10, 0, 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, ndim, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        rng = np.random.default_rng(7)
        shape = (23, 17, 11) if ndim == 3 else (41, 29)
        lv = rng.integers(0, 64, size=shape, dtype=np.int32)
        slab = slab_for(shape[0], world, rank)
        g = oracle.gather3d if ndim == 3 else oracle.gather2d
        # the rank holds only planes [r0, r1): emulate that by zeroing the rest
        local = np.full_like(lv, 0)
        local[slab.r0:slab.r1] = lv[slab.r0:slab.r1]
        q_in, q_out = g(local, 63, rows=slab.rows)
        h = torch.from_numpy(np.concatenate([q_in, q_out]).view(np.int64).copy())
        all_reduce_hist(h)
        full_in, full_out = g(lv, 63)
        ok = np.array_equal(h.numpy().view(np.uint64), np.concatenate([full_in, full_out]))
        result[rank] = int(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ndim", [2, 3])
def test_two_rank_allreduce_matches_single_process(ndim):
    world = 2
    ctx = mp.get_context("spawn")
    result = ctx.Array("i", [0] * world)
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ndim, result)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert list(result) == [1] * world
