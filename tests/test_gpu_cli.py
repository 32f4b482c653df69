"""The package CLI (python -m paper_2311_11740_b200 ...) on the GPU, byte for
byte against the reference CLI's output on the same seeded inputs
(tests/golden/cli/, made by tests/golden/gen_cli_golden.py from
/root/reference/pkg/src/fieldtopo/cli.py; cases in tests/cli_cases.py)."""
import contextlib
import io
from pathlib import Path

import pytest

from cli_cases import CASES, FILES

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden" / "cli"


@pytest.fixture(scope="module")
def files(tmp_path_factory):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2311_11740_b200 as ft
    tmp = tmp_path_factory.mktemp("cli")
    for name, (kind, dims, dist, seed, M, element) in FILES.items():
        f = ft.random_field(dims, dist, seed, M)
        p = tmp / name
        if kind == "bmp":
            ft.write_bmp(p, f)
        else:
            ft.write_raw_volume(p, f, element)
            if kind == "raw+sidecar":
                ft.write_sidecar(p, dims, element, M)
    return str(tmp)


def _run(argv, tmp):
    from paper_2311_11740_b200.cli import main
    argv = [a.replace("{tmp}", tmp) for a in argv]
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        code = main(argv)
    out = buf.getvalue()
    for a in argv:
        if a.endswith(".json") and a.startswith(tmp):
            out = Path(a).read_text()
    return code, out


@pytest.mark.parametrize("name", sorted(CASES))
def test_cli_matches_reference(files, name):
    code, out = _run(CASES[name], files)
    assert code == 0
    assert out == (GOLD / f"{name}.txt").read_text()


def test_cli_workers_and_devices_invariant(files):
    base = CASES["bmp_ec_perim"]
    outs = {_run(base + ["--workers", w], files)[1] for w in ("1", "8")}
    outs.add(_run(base + ["--devices", "cuda:0"], files)[1])
    assert len(outs) == 1


def test_cli_bench_runs(files, capsys):
    for path in ("map", "fused"):
        code, out = _run(["bench", "--generate", "64x48x40", "--repeats", "2", "--descriptor", "ec",
                          "--path", path, "--sweep-workers", "1,2"], files)
        assert code == 0
        lines = out.strip().splitlines()
        assert lines[0].startswith("bench: 64x48x40 cells=122880 repeats=2 descriptors=ec")
        assert lines[1].startswith("workers=1:") and "MV/s" in lines[1] and "speedup 1.00" in lines[1]
        assert lines[2].startswith("workers=2:")


def test_cli_connectivity_mismatch_exit_1(files):
    code, _ = _run(["curve", "--generate", "5x5", "--connectivity", "26"], files)
    assert code == 1
