"""Write BMP fixtures with the REFERENCE's own writer (run in the build
container, where /root/reference exists; the outputs are committed):
    NUMBA_CACHE_DIR=/tmp/nb PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_bmp_golden.py"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import fieldtopo as ref  # noqa: E402

OUT = Path(__file__).resolve().parent / "bmp"
OUT.mkdir(exist_ok=True)
rng = np.random.default_rng(31)
for name, shape in (("odd_7x5", (5, 7)), ("w8_8x3", (3, 8)), ("one_1x1", (1, 1))):
    lv = rng.integers(0, 256, size=shape).astype(np.int32)
    ref.write_bmp(OUT / f"{name}.bmp", ref.Field2D(lv, 255))
    np.save(OUT / f"{name}.npy", lv)
    assert np.array_equal(ref.read_bmp(OUT / f"{name}.bmp").values, lv)
print("wrote", sorted(p.name for p in OUT.iterdir()))
