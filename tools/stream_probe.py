"""End-to-end streaming throughput of the low-memory path by source kind:
pinned torch tensor (DMA straight from its pages), pageable numpy array and
raw f32 file (page cache) staged by the engine's host threads.  Same field
(1024 x 1024 x 2048 f32 = 8 GiB), descriptor_curves(ec, surface-area, volume),
curves equal across sources.   python tools/stream_probe.py"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2311_11740_b200 as ft  # noqa: E402
from paper_2311_11740_b200 import synth  # noqa: E402

dev = torch.device("cuda", 0)
shape = (1024, 1024, 2048)
x = synth.grf_slab(shape, 3.0, 7, (0, shape[0]), dev)
synth.normalise_(x, x.min(), x.max())
pinned = torch.empty(shape, dtype=torch.float32, pin_memory=True)
pinned.copy_(x)
host = pinned.numpy().copy()
del x
torch.cuda.empty_cache()
path = Path(os.environ.get("TMPDIR", "/tmp")) / "stream_probe.f32"
host.tofile(path)
tabs = [ft.builtin_weights(d, "26C") for d in ("ec", "surface-area", "volume")]
out, ref = {}, None
srcs = {"pinned_tensor": lambda: ft.ArraySource(pinned, 511, value_range=(0.0, 1.0)),
        "numpy_pageable": lambda: ft.ArraySource(host, 511, value_range=(0.0, 1.0)),
        "raw_f32_file": lambda: ft.open_raw_lowmem(path, (shape[1], shape[0], shape[2]), "f32", 511, (0.0, 1.0))}
for name, mk in srcs.items():
    times = []
    for it in range(3):
        src = mk()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        curves = np.stack([c.numerators for c in ft.descriptor_curves(src, tabs, chunk_bytes=512 << 20)])
        times.append(time.perf_counter() - t0)
        if hasattr(src, "close"):
            src.close()
    ref = curves if ref is None else ref
    s = min(times[1:])
    out[name] = {"GB_per_s": round(host.nbytes / s / 1e9, 2), "Gvox_per_s": round(host.size / s / 1e9, 3),
                 "curves_equal": bool(np.array_equal(curves, ref)), "staging_threads": min(16, os.cpu_count())}
path.unlink()
print(json.dumps({"field": list(shape), "bytes": host.nbytes, "sources": out}))
