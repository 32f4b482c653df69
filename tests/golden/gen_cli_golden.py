"""Golden CLI outputs from the REFERENCE command line (fieldtopo.cli.main,
/root/reference/pkg/src/fieldtopo/cli.py), for tests/test_gpu_cli.py.

Run in the build container only (reads /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/gen_cli_golden.py

Inputs are seeded: --generate fields, or files the reference writes from
random_field (BMP, raw u8 + sidecar, raw u16); the GPU test writes the same
files with the package's own writers.  Outputs land in tests/golden/cli/.
"""
import contextlib
import io
import os
import sys
import tempfile
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True
sys.path.insert(0, os.environ.get("FIELDTOPO_REF", "/root/reference/pkg/src"))

import fieldtopo as ft  # noqa: E402
from fieldtopo.cli import main  # noqa: E402

OUT = Path(__file__).resolve().parent / "cli"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from cli_cases import CASES, FILES  # noqa: E402


def write_files(tmp):
    for name, (kind, dims, dist, seed, M, element) in FILES.items():
        f = ft.random_field(dims, dist, seed, M)
        p = Path(tmp) / name
        if kind == "bmp":
            ft.write_bmp(p, f)
        else:
            ft.write_raw_volume(p, f, element)
            if kind == "raw+sidecar":
                ft.write_sidecar(p, dims, element, M)


def run(argv, tmp):
    argv = [a.replace("{tmp}", tmp) for a in argv]
    buf, err = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(buf), contextlib.redirect_stderr(err):
        code = main(argv)
    out = buf.getvalue()
    for a in argv:
        if a.endswith(".json") and a.startswith(tmp):
            out = Path(a).read_text()
    return code, out


if __name__ == "__main__":
    OUT.mkdir(exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        write_files(tmp)
        for name, argv in CASES.items():
            code, out = run(argv, tmp)
            assert code == 0, (name, code)
            (OUT / f"{name}.txt").write_text(out)
            print(name, len(out))
