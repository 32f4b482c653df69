"""Profiling driver: build a synthetic field on cuda:0 and launch the hot
kernels a few times (for ncu / timing).
    python tools/prof_run.py [c4a|c5|small] [reps] [map|lattice|both]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2311_11740_b200 as ft  # noqa: E402
from paper_2311_11740_b200 import engine, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4a"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kind = sys.argv[3] if len(sys.argv) > 3 else "both"
shape, sigma, M = {"c4a": ((512, 512, 512), 3.0, 255), "c5": ((2048, 2048, 2048), 4.0, 511),
                   "small": ((256, 256, 256), 3.0, 255)}[cfg]
dev = torch.device("cuda", 0)
x = synth.grf_slab(shape, sigma, 2311, (0, shape[0]), dev)
synth.normalise_(x, x.min(), x.max())
q = ft.quant.QuantSpec.for_range(0.0, 1.0, M)
torch.cuda.synchronize()
for name in (("map", "lattice") if kind == "both" else (kind,)):
    h = engine.new_hist(3, M, dev) if name == "map" else engine.new_lattice_hist(3, M, dev)
    launch = engine.launch_hist if name == "map" else engine.launch_lattice
    for r in range(reps):
        h.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        launch(3, x, shape, M, q, hist=h)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{cfg} {name} rep {r}: {dt * 1e3:.3f} ms  {x.numel() / dt / 1e9:.1f} Gvox/s")
