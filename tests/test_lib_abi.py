"""CPU-side checks of the C-ABI boundary: libf3d.so loads and exports every
symbol declared in include/f3d.h, and the ctypes table matches the header.
No compute calls (no GPU here)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "f3d.h")
LIB = os.path.join(ROOT, "paper_2412_16481_b200", "libf3d.so")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(f3d_\w+)\s*\(", src)))


@pytest.mark.skipif(not os.path.exists(LIB), reason="libf3d.so not built (run __graft_entry__.build())")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    names = declared()
    assert len(names) >= 10
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.f3d_abi_version() == 1


def test_ctypes_table_covers_header():
    from paper_2412_16481_b200 import _lib
    assert set(declared()) == set(_lib.SIGNATURES), set(declared()) ^ set(_lib.SIGNATURES)


@pytest.mark.skipif(not os.path.exists(LIB), reason="libf3d.so not built")
def test_config_errors_need_no_gpu():
    """Argument validation happens before any CUDA call."""
    lib = ctypes.CDLL(LIB)
    assert lib.f3d_scatter_rows(None, None, ctypes.c_int64(4), ctypes.c_int64(6), None, None,
                                None) == 1
    lib.f3d_psh_workspace_size.restype = ctypes.c_size_t
    assert lib.f3d_psh_workspace_size(ctypes.c_int64(1000), 1, 40) > 0


def test_launch_table_is_consistent():
    from paper_2412_16481_b200 import _lib
    assert set(_lib.KERNELS_PER_CALL) <= set(_lib.SIGNATURES)
    assert all(isinstance(v, int) and v >= 0 for v in _lib.KERNELS_PER_CALL.values())
