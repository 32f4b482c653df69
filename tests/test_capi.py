"""The C-ABI library loads and exports every symbol include/*.h declares
(no compute calls: this runs without a GPU)."""
import ctypes
import re
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    syms = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        syms |= set(re.findall(r"\b(ft_[a-z0-9_]+)\s*\(", text))
    return syms


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("ft_hist2d", "ft_hist3d", "ft_finalize", "ft_curves", "ft_quantize", "ft_minmax"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2311_11740_b200 import _lib
    L = _lib.load()
    for s in declared_symbols():
        assert hasattr(L, s), s
    assert set(_lib.EXPORTS) == declared_symbols()


def test_library_is_sm100a_only():
    import subprocess
    from paper_2311_11740_b200 import build
    out = subprocess.run(["cuobjdump", "--list-elf", str(build.LIB)], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_\d+a?", out))
    assert arches == {"sm_100a"}, arches


def test_argument_errors_without_gpu():
    from paper_2311_11740_b200 import _lib
    L = _lib.load()
    win = _lib.ft_window(None, 0, 0, 0, 1, 0)
    q = _lib.ft_quant(0, 0, 0.0, 0.0, None)
    # bad shapes / ranges are rejected before any CUDA call
    assert L.ft_hist3d(ctypes.byref(win), 0, 4, 4, 0, 1, ctypes.byref(q), 5, None, None) == 1
    assert L.ft_hist2d(ctypes.byref(win), 4, 4, 0, 9, ctypes.byref(q), 5, None, None) == 1
    assert L.ft_finalize(4, 5, 1, None, None, None, 0, None, None, None) == 1
    w = np.zeros(21, np.int64)
    out = np.zeros(40, np.int64)
    assert L.ft_class_weights(3, w.ctypes.data, out.ctypes.data) == 0
    assert L.ft_version().startswith(b"fieldtopo-b200")
