"""The C-ABI boundary: libigb.so loads and exports every symbol include/igb.h declares.

No compute calls here (no GPU in the CPU suite); igb_create must fail cleanly
without a device, and the Python binding must refuse to fall back to the CPU.
"""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "igb.h")
LIB = os.path.join(ROOT, "paper_1902_01818_b200", "libigb.so")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(igb_[a-z0-9_]+)\s*\(", text)))


def _lib():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    return ctypes.CDLL(LIB)


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("igb_create", "igb_set_level_matrix", "igb_set_prolongation", "igb_set_gs",
                     "igb_scms_add_interior", "igb_scms_add_piece", "igb_set_coarse_lu",
                     "igb_cycle", "igb_pcg", "igb_pcg_device", "igb_op"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = _lib()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_signatures_cover_header():
    from paper_1902_01818_b200 import _lib as binding
    assert set(declared_functions()) <= set(binding.SIGNATURES)


def test_version_and_null_context_errors():
    lib = _lib()
    lib.igb_version.restype = ctypes.c_int
    assert lib.igb_version() >= 1
    lib.igb_set_num_levels.argtypes = [ctypes.c_void_p, ctypes.c_int]
    assert lib.igb_set_num_levels(None, 3) < 0


def test_no_cpu_fallback_without_device():
    from paper_1902_01818_b200 import _lib as binding
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a CUDA device is present")
    except ImportError:
        pass
    with pytest.raises(RuntimeError):
        binding.Context(0)
