"""CLI argument handling that fails before any GPU work (CPU): the
reference's exit codes (cli.py:250-281) -- 1 for usage and input errors."""
import pytest

from paper_2311_11740_b200.cli import build_parser, main


@pytest.mark.parametrize("argv", [
    [],                                                   # no command
    ["frobnicate"],                                       # unknown command
    ["curve"],                                            # neither --input nor --generate
    ["curve", "--generate", "6"],                         # bad dims
    ["curve", "--generate", "6x0"],                       # zero extent
    ["curve", "--generate", "2x3x4x5"],                   # too many dims
    ["curve", "--generate", "6x4", "--input", "a.bmp"],   # both
    ["curve", "--generate", "6x4", "--low-memory"],       # low memory on a generated field
    ["curve", "--input", "field.xyz"],                    # unknown suffix
    ["curve", "--input", "v.raw"],                        # raw without dims or sidecar
    ["curve", "--input", "v.raw", "--dims", "4x4"],       # raw dims must be 3D
    ["curve", "--input", "/nonexistent/x.bmp"],           # unreadable file (OSError)
    ["bench", "--generate", "4x4", "--repeats", "x"],     # bad int
])
def test_usage_errors_exit_1(argv, tmp_path, monkeypatch, capsys):
    monkeypatch.chdir(tmp_path)
    assert main(argv) == 1


def test_parser_defaults():
    a = build_parser().parse_args(["bench", "--generate", "8x8"])
    assert (a.repeats, a.workers, a.max_level, a.path, a.dist) == (5, 1, 255, "map", "uniform")


def test_internal_consistency_failure_exits_2(tmp_path, monkeypatch, capsys):
    """A ClassificationError from the gather (reference contrib3d.py:425-426)
    is reported as an internal consistency failure with exit code 2
    (reference cli.py:271-273, pkg/tests/test_cli.py:139-150)."""
    import numpy as np

    import paper_2311_11740_b200 as ft
    from paper_2311_11740_b200 import cli

    def boom(source, workers, **kw):
        raise ft.ClassificationError("q-table miss")

    monkeypatch.setattr(cli, "gather_2d_parallel", boom)
    p = tmp_path / "x.bmp"
    ft.write_bmp(p, ft.Field2D(np.zeros((1, 1), np.int32), 255))
    assert main(["curve", "--input", str(p)]) == 2
    assert "internal consistency" in capsys.readouterr().err
