"""The C-ABI library builds, loads without a GPU and exports every symbol
declared in include/*.h (no compute calls here)."""

import ctypes
import glob
import os
import re

import pytest

from paper_2009_12638_b200 import _lib
from paper_2009_12638_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
        for m in re.finditer(r"\b(bs_[a-z_0-9]+)\s*\(", text):
            names.add(m.group(1))
    return sorted(names)


def test_header_declares_entry_points():
    names = declared_symbols()
    assert "bs_cg_begin" in names and "bs_stencil_apply" in names and len(names) >= 12


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(build())
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_ctypes_signatures_cover_header():
    assert set(declared_symbols()) == set(_lib._SIGS)


def test_abi_version_and_error_path_without_gpu():
    lib = _lib.load()
    assert lib.bs_abi_version() == 2
    # argument validation happens before any CUDA call
    assert lib.bs_ctx_create(0, 0, None, 0, None) == -1
    assert b"bad arguments" in lib.bs_last_error()
    with pytest.raises(Exception):
        _lib.check(-1)


def test_struct_layout_matches_header():
    # bs_block_desc: 10 int32 (+4 pad) + 5 ptr + 6 ptr + ptr + int32 (+4 pad)
    assert ctypes.sizeof(_lib.BlockDesc) == 40 + 8 * 12 + 8
    assert ctypes.sizeof(_lib.BlockReport) == 16 + 6 * 8 + 8
