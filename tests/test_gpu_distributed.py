"""The product's multi-rank entry points executed with the real CUDA kernels
(reference _parallel.py:8-33; acceptance c5, pkg/tests/test_acceptance.py:
288-304: every partition gives the identical map).

World sizes 2 and 3, one process per rank, gloo with CUDA tensors (this pool
has one GPU per box, so every rank uses cuda:0; ranks never wait on each
other's kernels -- the only exchange is the histogram all-reduce).  Each rank
holds ONLY its slab's planes (``distributed.slab_for``: uneven splits of
H + 1 vertex rows) and calls ``descriptor_curves_distributed`` (fused line /
lattice kernels) and ``gather_distributed`` (map kernel + finalize); every
rank's result must equal the single-GPU result and the oracle bit for bit."""
import os
import pickle
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _field(ndim):
    rng = np.random.default_rng(21 + ndim)
    if ndim == 3:
        from scipy.ndimage import gaussian_filter
        x = gaussian_filter(rng.standard_normal((29, 37, 70)).astype(np.float32), 1.5, mode="wrap")
    else:
        from scipy.ndimage import gaussian_filter
        x = gaussian_filter(rng.standard_normal((61, 133)).astype(np.float32), 2.0, mode="wrap")
    return ((x - x.min()) / (x.max() - x.min())).astype(np.float32)


def _tables(ft, ndim):
    if ndim == 3:
        return [ft.builtin_weights(d, "26C") for d in ("ec", "surface-area", "volume", "perimeter")]
    return [ft.builtin_weights(*t) for t in (("ec", "8C"), ("ec", "4C"), ("perimeter", "8C"), ("area", "8C"))]


def _rank_main(rank, world, port, ndim, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2311_11740_b200 as ft
        from paper_2311_11740_b200.distributed import descriptor_curves_distributed, gather_distributed, slab_for
        x = _field(ndim)
        M = 255
        slab = slab_for(x.shape[0], world, rank)
        local = torch.from_numpy(np.ascontiguousarray(x[slab.r0:slab.r1])).to("cuda:0")  # this rank's planes only
        tabs = _tables(ft, ndim)
        curves = descriptor_curves_distributed(local, x.shape, M, tabs[:3] if ndim == 3 else tabs,
                                               value_range=(0.0, 1.0))
        cmap = gather_distributed(local, x.shape, M, value_range=(0.0, 1.0))
        with open(os.path.join(out_dir, f"r{rank}.pkl"), "wb") as fh:
            pickle.dump({"curves": [c.numerators for c in curves], "q_in": cmap.q_in, "q_out": cmap.q_out,
                         "slab": (slab.v0, slab.v1, slab.r0, slab.r1)}, fh)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ndim", [2, 3])
@pytest.mark.parametrize("world", [2, 3])
def test_distributed_entry_points_on_gpu(ndim, world, orc, tmp_path):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_11740_b200 as ft
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, ndim, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    x = _field(ndim)
    M = 255
    g = orc.gather3d if ndim == 3 else orc.gather2d
    q_in, q_out = g(x, M, value_range=(0.0, 1.0), workers=8)
    tabs = _tables(ft, ndim)
    single = ft.descriptor_curves(ft.DeviceSource(torch.from_numpy(x).cuda(), M, value_range=(0.0, 1.0)),
                                  tabs[:3] if ndim == 3 else tabs)
    slabs = []
    for r in range(world):
        with open(tmp_path / f"r{r}.pkl", "rb") as fh:
            res = pickle.load(fh)
        slabs.append(res["slab"][:2])
        assert np.array_equal(res["q_in"], q_in) and np.array_equal(res["q_out"], q_out), r
        for c, s, t in zip(res["curves"], single, tabs):
            assert np.array_equal(c, s.numerators), (r, t.descriptor)
            assert np.array_equal(c, orc.descriptor_numerators(q_in, q_out, M, t.eighths)), (r, t.descriptor)
    # the slabs are an uneven split of all H + 1 vertex rows
    assert slabs[0][0] == 0 and slabs[-1][1] == x.shape[0] + 1
    assert all(a[1] == b[0] for a, b in zip(slabs, slabs[1:]))
