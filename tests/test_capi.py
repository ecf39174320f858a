"""The C-ABI library loads and exports every entry point include/*.h declares
(CPU-only: no compute calls)."""

import ctypes
import os
import re

import pytest

from paper_2505_14741_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "parastep_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ps_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_binding():
    assert set(_declared()) == set(_lib.EXPORTED)


def test_library_exports_every_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in _declared() if not hasattr(lib, s)]
    assert not missing, missing
    assert _lib.load().ps_version() == 1


def test_no_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    from paper_2505_14741_b200.numerics import draw_normal

    with pytest.raises(_lib.NativeLibraryError):
        draw_normal(1, 2, 8)
