"""One-off randomized differential run on the GPU: random shapes, dtypes, level
counts and value ranges through the public API (gather_* maps and
descriptor_curves) against the pinned oracle, bit-exact.
    python tools/gpu_fuzz.py [cases] [seed]"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2311_11740_b200 as ft  # noqa: E402
from oracle import oracle as orc  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
MS = [1, 2, 3, 7, 63, 100, 255, 256, 511, 600, 601, 602, 763, 764, 1023, 1100, 1380, 1500, 2047, 2265, 2300, 2400,
      2728, 2729, 4095]
T3 = [("ec", "26C"), ("perimeter", "26C"), ("surface-area", "26C"), ("volume", "26C")]
T2 = [("ec", "8C"), ("ec", "4C"), ("perimeter", "8C"), ("area", "8C")]
fails = 0
t0 = time.time()
for case in range(N):
    ndim = int(rng.integers(2, 4))
    M = int(rng.choice(MS))
    if ndim == 2:
        shape = (int(rng.integers(1, 400)), int(rng.integers(1, 1500)))
    else:
        shape = (int(rng.integers(1, 60)), int(rng.integers(1, 200)), int(rng.integers(1, 400)))
    kind = rng.choice(["i32", "u8", "u16", "u16ri", "u16rf", "u8r", "f32p", "f32t", "f32n"])
    vr = None
    if kind == "i32":
        x = rng.integers(0, M + 1, size=shape, dtype=np.int32)
    elif kind == "u8":
        M = min(M, 255)
        x = rng.integers(0, M + 1, size=shape).astype(np.uint8)
    elif kind == "u16":
        x = rng.integers(0, M + 1, size=shape).astype(np.uint16)
    elif kind in ("u16ri", "u16rf"):
        x = rng.integers(0, 65536, size=shape).astype(np.uint16)
        lo = int(rng.integers(0, 30000))
        hi = lo + int(rng.integers(1, 35000))
        vr = (float(lo), float(hi)) if kind == "u16ri" else (lo + 0.37, hi + 0.61)
    elif kind == "u8r":
        x = rng.integers(0, 256, size=shape).astype(np.uint8)
        lo = int(rng.integers(0, 100))
        vr = (float(lo), float(lo + int(rng.integers(1, 155))))
    else:
        x = rng.random(shape, dtype=np.float32)
        if rng.random() < 0.3:  # out-of-range values and exact thresholds
            x = (x * 1.4 - 0.2).astype(np.float32)
        vr = {"f32p": (0.0, float(rng.choice([0.5, 1.0, 2.0]))), "f32t": (0.13, 0.91), "f32n": (0.9, 0.1)}[kind]
    levels = x.astype(np.int32) if vr is None else orc.quantize_with_range(x, vr[0], vr[1], M)
    gather = orc.gather2d if ndim == 2 else orc.gather3d
    q_in, q_out = gather(levels, M, workers=8)
    if kind == "i32":
        src = (ft.Field2D if ndim == 2 else ft.Field3D)(x, M)
    else:
        xt = torch.from_numpy(x.astype(np.int32)).to(torch.uint16).cuda() if x.dtype == np.uint16 else torch.from_numpy(x).cuda()
        src = ft.DeviceSource(xt, M, value_range=vr)
    ok = True
    try:
        m = (ft.gather_2d_serial if ndim == 2 else ft.gather_3d_serial)(src)
        ok &= bool(np.array_equal(m.q_in, q_in) and np.array_equal(m.q_out, q_out))
        tabs = [ft.builtin_weights(*t) for t in (T2 if ndim == 2 else T3)]
        for c, t in zip(ft.descriptor_curves(src, tabs), tabs):
            ok &= bool(np.array_equal(c.numerators, orc.descriptor_numerators(q_in, q_out, M, t.eighths)))
    except Exception as e:  # noqa: BLE001
        ok = False
        print("EXC", repr(e))
    if not ok:
        fails += 1
        print("FAIL", case, ndim, shape, kind, M, vr)
print(f"{N} cases, {fails} failures, {time.time() - t0:.1f} s")
sys.exit(1 if fails else 0)
