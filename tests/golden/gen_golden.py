"""Generate golden vectors for the oracle pin by importing the REFERENCE.

Run in the build container only (it reads /root/reference, which does not
exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/gen_golden.py

Writes tests/golden/golden.npz.  Every input is produced here from a seeded
generator (nothing is copied from the reference's own test data); every output
is computed by the reference package's public functions:
quantize_with_range (fields.py:20-33), gather_2d_serial / gather_3d_serial
(contrib2d.py:264, contrib3d.py:430), accumulate_vertex_2d/3d
(contrib2d.py:139, contrib3d.py:220), classify_config + pair_classes
(contrib3d.py:76-135), builtin_weights + descriptor_curve
(descriptors.py:109-178).
"""
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True
REF = os.environ.get("FIELDTOPO_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import numpy as np  # noqa: E402
import fieldtopo as ft  # noqa: E402
from fieldtopo.contrib2d import TYPE_NAMES_2D  # noqa: E402
from fieldtopo.contrib3d import TYPE_NAMES_3D  # noqa: E402

OUT = Path(__file__).resolve().parent / "golden.npz"
g = {}

# ---- quantize_with_range --------------------------------------------------
rng = np.random.default_rng(1234)
qcases = [(0.0, 1.0, 99), (0.0, 1.0, 255), (0.0, 1.0, 511), (-3.7, 4.2, 1023),
          (0.25, 0.75, 7), (2.0, 2.0, 255), (1.0, 0.0, 63)]
for n, (lo, hi, M) in enumerate(qcases):
    x = np.concatenate([
        rng.random(4000, dtype=np.float32) * (hi - lo) * 1.2 + lo - 0.1 * (hi - lo),
        rng.standard_normal(1000).astype(np.float32) * 3,
        np.array([lo, hi, -np.inf, np.inf, 0.0, -0.0, 1e30, -1e30], np.float32),
        # exact half-way points of the float64 formula (round-half-up pins)
        (np.float32(lo) + (np.arange(0, M + 1, dtype=np.float64) + 0.5)
         * (hi - lo) / M).astype(np.float32) if hi != lo else np.zeros(1, np.float32),
    ]).astype(np.float32)
    g[f"quant{n}_x"] = x
    g[f"quant{n}_params"] = np.array([lo, hi, M], np.float64)
    g[f"quant{n}_levels"] = ft.quantize_with_range(x, lo, hi, M)
u16 = rng.integers(0, 65536, 5000).astype(np.uint16)
u16[:2] = (0, 65535)
g["quant_u16_x"] = u16
g["quant_u16_levels"] = ft.quantize(u16, 1023)
g["n_quant"] = np.array(len(qcases))

# ---- 2D contribution maps + curves -----------------------------------------
cases2d = [((6, 5), "uniform", 0, 12), ((9, 3), "uniform", 1, 3), ((1, 7), "uniform", 2, 2),
           ((4, 4), "uniform", 3, 0), ((11, 8), "uniform", 4, 255), ((12, 10), "uniform", 5, 1),
           ((33, 17), "normal", 1, 63), ((1, 1), "uniform", 6, 9), ((7, 1), "normal", 7, 5),
           ((64, 48), "normal", 8, 255), ((70, 3), "uniform", 9, 1)]
tables2d = [("ec", "8C"), ("ec", "4C"), ("perimeter", "8C"), ("area", "8C")]
for n, (dims, dist, seed, M) in enumerate(cases2d):
    f = ft.random_field(dims, dist, seed=seed, max_level=M)
    m = ft.gather_2d_serial(f)
    g[f"f2d{n}_levels"] = f.values.copy()
    g[f"f2d{n}_M"] = np.array(M)
    g[f"f2d{n}_qin"] = m.q_in
    g[f"f2d{n}_qout"] = m.q_out
    g[f"f2d{n}_curves"] = np.stack([ft.descriptor_curve(m, ft.builtin_weights(*t)).numerators
                                    for t in tables2d])
g["n_f2d"] = np.array(len(cases2d))

# Config-1 shape: 256x256 float32 Uniform[0,1) quantized to M=99 on [0,1].
x1 = np.random.default_rng(2311).random((256, 256), dtype=np.float32)
lv1 = ft.quantize_with_range(x1, 0.0, 1.0, 99)
m1 = ft.gather_2d_serial(ft.Field2D(lv1, 99))
g["c1_x"] = x1
g["c1_qin"] = m1.q_in
g["c1_qout"] = m1.q_out
g["c1_curves"] = np.stack([ft.descriptor_curve(m1, ft.builtin_weights(*t)).numerators
                           for t in tables2d])

# ---- 3D contribution maps + curves -----------------------------------------
cases3d = [((3, 2, 4), "uniform", 0, 9), ((2, 2, 2), "uniform", 1, 1), ((5, 1, 3), "uniform", 2, 4),
           ((4, 3, 2), "uniform", 3, 255), ((4, 3, 5), "normal", 7, 6), ((9, 8, 6), "normal", 4, 31),
           ((1, 1, 1), "uniform", 5, 3), ((1, 1, 9), "uniform", 6, 2), ((13, 11, 7), "uniform", 8, 1),
           ((12, 10, 14), "normal", 9, 255)]
tables3d = [("ec", "26C"), ("perimeter", "26C"), ("surface-area", "26C"), ("volume", "26C")]
for n, (dims, dist, seed, M) in enumerate(cases3d):
    f = ft.random_field(dims, dist, seed=seed, max_level=M)
    m = ft.gather_3d_serial(f)
    g[f"f3d{n}_levels"] = f.values.copy()
    g[f"f3d{n}_M"] = np.array(M)
    g[f"f3d{n}_qin"] = m.q_in
    g[f"f3d{n}_qout"] = m.q_out
    g[f"f3d{n}_curves"] = np.stack([ft.descriptor_curve(m, ft.builtin_weights(*t)).numerators
                                    for t in tables3d])
g["n_f3d"] = np.array(len(cases3d))

# Float 3D volume quantized on [0,1] with M=255 (config-4a style, small).
x4 = np.random.default_rng(5120).random((20, 18, 16), dtype=np.float32)
lv4 = ft.quantize_with_range(x4, 0.0, 1.0, 255)
m4 = ft.gather_3d_serial(ft.Field3D(lv4, 255))
g["c4_x"] = x4
g["c4_qin"] = m4.q_in
g["c4_qout"] = m4.q_out

# ---- single-vertex known answers -------------------------------------------
vr = np.random.default_rng(77)
v2 = vr.integers(0, 6, size=(300, 4))
v2[:, :][vr.random((300, 4)) < 0.2] = 6  # sentinel M+1 for M=5
acc2_in, acc2_out = [], []
for row in v2:
    c = ft.ContributionMap2D.zeros(1, 1, 5)
    ft.accumulate_vertex_2d(ft.VertexNeighborhood2D(tuple(int(t) for t in row)), c)
    acc2_in.append(c.q_in)
    acc2_out.append(c.q_out)
g["acc2_vals"] = v2
g["acc2_qin"] = np.stack(acc2_in)
g["acc2_qout"] = np.stack(acc2_out)
v3 = vr.integers(0, 5, size=(600, 8))
v3[vr.random((600, 8)) < 0.2] = 5  # sentinel for M=4
acc3_in, acc3_out = [], []
for row in v3:
    c = ft.ContributionMap3D.zeros(1, 1, 1, 4)
    ft.accumulate_vertex_3d(ft.VertexNeighborhood3D(tuple(int(t) for t in row)), c)
    acc3_in.append(c.q_in)
    acc3_out.append(c.q_out)
g["acc3_vals"] = v3
g["acc3_qin"] = np.stack(acc3_in)
g["acc3_qout"] = np.stack(acc3_out)

# ---- classification of every 3D mask (stage n = popcount) -------------------
cls = np.full(256, -1, np.int64)
for mask in range(1, 256):
    act = [s for s in range(8) if mask >> s & 1]
    emp = [s for s in range(8) if not mask >> s & 1]
    n = len(act)
    cls[mask] = ft.classify_config(n, ft.pair_classes(act if n <= 4 else emp))
g["classify3d"] = cls

# ---- weight tables ----------------------------------------------------------
g["w2d"] = np.array([ft.builtin_weights(*t).eighths for t in tables2d], np.int64)
g["w3d"] = np.array([ft.builtin_weights(*t).eighths for t in tables3d], np.int64)
g["type_names_2d"] = np.array(TYPE_NAMES_2D)
g["type_names_3d"] = np.array(TYPE_NAMES_3D)

np.savez_compressed(OUT, **g)
print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(g)} arrays)")
