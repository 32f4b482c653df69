"""Build A/B variants of the benchmark path's translation unit (ft_lines_f32p.cu:
f32 / FT_Q_POW2) linked with the other objects of the main build:  python tools/dev/variants.py name="-DX=1 -DY=2" ...
Each lands in variants/<name>/libfieldtopo_b200.so (use with FT_DEV_LIB=... python tools/prof_run.py; dev A/B only)."""
import concurrent.futures as cf
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2311_11740_b200 import build as b  # noqa: E402

UNIT = "ft_lines_f32p"
if len(sys.argv) > 1 and sys.argv[1].startswith("--unit="):
    UNIT = sys.argv.pop(1).split("=", 1)[1]  # e.g. --unit=ft_lines2d
objs = [p for p in sorted(b.BUILD.glob("*.o")) if p.stem != UNIT]


def one(spec):
    name, flags = spec.split("=", 1)
    out = ROOT / "variants" / name
    out.mkdir(parents=True, exist_ok=True)
    obj = out / f"{UNIT}.o"
    cmd = [b.nvcc(), *b.ARCH, *b.NVCC_FLAGS, *flags.split(), "-Xptxas", "-v", "-c",
           str(b.CSRC / f"{UNIT}.cu"), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        return f"{name}: FAILED\n{r.stderr[-2000:]}"
    info = [l for l in r.stderr.splitlines() if "registers" in l or "spill" in l]
    r2 = subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-o", str(out / "libfieldtopo_b200.so"), str(obj),
                         *map(str, objs)], capture_output=True, text=True)
    return f"{name}: {'ok' if not r2.returncode else r2.stderr[-500:]}  " + " | ".join(info[-4:])


with cf.ThreadPoolExecutor(8) as ex:
    for line in ex.map(one, sys.argv[1:]):
        print(line)
