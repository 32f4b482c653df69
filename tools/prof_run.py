"""Profiling driver: build a synthetic field on cuda:0 and launch the hot
kernels a few times (for ncu / timing).
    python tools/prof_run.py [c4a|c4b|c5|small|c2|c3] [reps] [map|lattice|lines|both|all]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_11740_b200 as ft  # noqa: E402
from paper_2311_11740_b200 import engine, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4a"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kind = sys.argv[3] if len(sys.argv) > 3 else "both"
dev = torch.device("cuda", 0)
batch, bstride = 1, 0
if cfg in ("c4a", "c5", "small"):
    shape, sigma, M = {"c4a": ((512, 512, 512), 3.0, 255), "c5": ((2048, 2048, 2048), 4.0, 511),
                       "small": ((256, 256, 256), 3.0, 255)}[cfg]
    x = synth.grf_slab(shape, sigma, 2311, (0, shape[0]), dev)
    synth.normalise_(x, x.min(), x.max())
    q = ft.quant.QuantSpec.for_range(0.0, 1.0, M)
elif cfg == "c4b":  # 1024 x 1024 x 256 u16 hyperspectral-like cube, auto-range quantize to 1024 levels
    shape, M = (1024, 1024, 256), 1023
    x = synth.grf_slab(shape, 3.0, 2311, (0, shape[0]), dev)
    synth.normalise_(x, x.min(), x.max())
    xi = torch.floor(x * 65535 + 0.5).to(torch.int32)
    lo, hi = float(xi.min()), float(xi.max())
    x = xi.to(torch.uint16)
    del xi
    q = ft.quant.QuantSpec.for_range(lo, hi, M)
elif cfg == "c2":
    shape, M = (8192, 8192), 255
    x = synth.grf_2d(shape, 4.0, 2311, dev)
    synth.normalise_(x, x.min(), x.max())
    q = ft.quant.QuantSpec.for_range(0.0, 1.0, M)
else:  # c3: 512 microscopy-like u8 images, 1024^2, sigma ~ U[1, 8]
    shape, M, batch = (1024, 1024), 255, 512
    sig = np.random.default_rng(2311).uniform(1.0, 8.0, batch)
    x = torch.empty((batch,) + shape, dtype=torch.uint8, device=dev)
    for b in range(batch):
        im = synth.grf_2d(shape, float(sig[b]), 2311 + b, dev)
        im = (im - im.min()) / (im.max() - im.min())
        x[b] = torch.floor(im * 255 + 0.5).to(torch.uint8)
    bstride = shape[0] * shape[1]
    q = ft.quant.QuantSpec.identity()
ndim = len(shape)
cells = x.numel()
torch.cuda.synchronize()
names = {"both": ("map", "lattice"), "all": ("map", "lattice", "lines")}.get(kind, (kind,))
for name in names:
    if name == "lines" and ndim != 3:
        continue
    for r in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if name == "map":
            engine.launch_hist(ndim, x, shape, M, q, batch=batch, batch_stride=bstride)
        elif name == "lines":
            engine.launch_lines(x, shape, M, q)
        else:
            engine.launch_lattice(ndim, x, shape, M, q, batch=batch, batch_stride=bstride)
        e1.record()
        torch.cuda.synchronize()
        dt = e0.elapsed_time(e1) / 1e3  # launches go to torch's current stream
        print(f"{cfg} {name} rep {r}: {dt * 1e3:.3f} ms  {cells / dt / 1e9:.1f} Gvox/s")
