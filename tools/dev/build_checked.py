"""Build the whole library with -DFT_BOUNDS_CHECK (every shared-memory
histogram update traps if it leaves its block) into variants/checked/, and
optionally run pytest against it:

    python tools/dev/build_checked.py            # build only
    python tools/dev/build_checked.py -m gpu -q  # build, then pytest with these args

compute-sanitizer is closed on the GPU pool; this is the substitute.  Dev only:
the package itself always loads paper_2311_11740_b200/_build."""
import concurrent.futures as cf
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2311_11740_b200 import build as b  # noqa: E402

OUT = ROOT / "variants" / "checked"
LIB = OUT / "libfieldtopo_b200.so"


def build():
    OUT.mkdir(parents=True, exist_ok=True)

    def one(src):
        obj = OUT / (src.stem + ".o")
        r = subprocess.run([b.nvcc(), *b.ARCH, *b.NVCC_FLAGS, "-DFT_BOUNDS_CHECK", "-c", str(src), "-o", str(obj)],
                           capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stderr[-3000:])
        return obj

    with cf.ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(one, b._sources()))
    r = subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-ldl"],
                       capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr[-3000:])
    for o in objs:
        o.unlink()
    return LIB


if __name__ == "__main__":
    if not LIB.exists() or "--rebuild" in sys.argv:
        print(build())
    args = [a for a in sys.argv[1:] if a != "--rebuild"]
    if args:
        b.LIB = LIB  # the package loads the checked library from here on
        from paper_2311_11740_b200 import _lib
        _lib.load(build_if_missing=False)
        import pytest
        rc = pytest.main([str(ROOT / "tests"), *args])
        maps = {line.split()[-1] for line in open("/proc/self/maps") if "libfieldtopo" in line}
        print("libfieldtopo mapped in this process:", sorted(maps))
        sys.exit(rc)
