"""The C-ABI library builds, loads on CPU and exports every entry point that
include/ldgb200.h declares (no compute calls without a GPU)."""

import ctypes
import re
from pathlib import Path

from paper_2205_07824_b200 import _lib
from paper_2205_07824_b200.build import build

HEADER = Path(__file__).resolve().parent.parent / "include" / "ldgb200.h"


def declared():
    txt = HEADER.read_text()
    return sorted(set(re.findall(r"\b(ldg_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_header_symbols():
    lib = ctypes.CDLL(str(build()))
    names = declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTED)
    assert lib.ldg_version() == 1


def test_table_struct_layout_matches_header():
    # 8 int32 + 5 pointers + 3*81 + 2*9 + 75 + 225 + 5 doubles
    assert ctypes.sizeof(_lib.LdgTables) == 8 * 4 + 5 * 8 + (3 * 81 + 18 + 75 + 225 + 5) * 8
