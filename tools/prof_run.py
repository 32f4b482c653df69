"""Profiling driver: build a synthetic field on cuda:0 and launch the hot
kernels a few times (for ncu / timing).
    python tools/prof_run.py [c1|c2|c3|c4a|c4b|c5|small] [reps] [map|lattice|lines|both|all]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import os  # noqa: E402

if os.environ.get("FT_DEV_LIB"):  # dev A/B only: load a variant build of the library
    from paper_2311_11740_b200 import _lib, build as _b  # noqa: E402
    _b.LIB = Path(os.environ["FT_DEV_LIB"]).resolve()
    _lib.load(build_if_missing=False)
import paper_2311_11740_b200 as ft  # noqa: E402
from paper_2311_11740_b200 import engine, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4a"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kind = sys.argv[3] if len(sys.argv) > 3 else "both"
dev = torch.device("cuda", 0)
cfg_d = synth.config_field(cfg if cfg != "small" else "c4a", dev) if cfg != "small" else None
if cfg == "small":
    shape, M = (256, 256, 256), 255
    x = synth.grf_slab(shape, 3.0, 2311, (0, 256), dev)
    synth.normalise_(x, x.min(), x.max())
    vr = (0.0, 1.0)
else:
    x, M, shape, vr = cfg_d["x"], cfg_d["M"], cfg_d["shape"], cfg_d["value_range"]
batch = cfg_d["batch"] if cfg_d else 1
bstride = shape[0] * shape[1] if batch > 1 else 0
if vr == "auto":
    vr = engine.minmax_device(x)
q = ft.quant.QuantSpec.for_range(vr[0], vr[1], M) if vr is not None else ft.quant.QuantSpec.identity()
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
