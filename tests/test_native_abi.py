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


def test_native_distance2_coloring_matches_reference_greedy():
    """ldg_color_distance2 == the reference's greedy on the squared graph
    (solver.py:355-378) on structured, periodic and simplex meshes."""
    import numpy as np
    from paper_2205_07824_b200 import meshgen
    from paper_2205_07824_b200.solver import (distance2_coloring, distance2_coloring_topology,
                                              element_neighbor_sets)
    for counts, kind, per in (([5, 4, 3], "hex", None), ([4, 4], "quad",
                                                         [(1, 2, (1.0, 0.0)), (3, 4, (0.0, 1.0))]),
                              ([3, 3, 2], "tet", None), ([6, 5], "tri", None)):
        nd = len(counts)
        mesh = meshgen.generate_structured([(0.0, 1.0)] * nd, counts, kind)
        topo = meshgen.build_face_topology(mesh, per)
        ne = mesh.connectivity.shape[0]
        want = distance2_coloring(element_neighbor_sets(topo, ne))
        assert np.array_equal(distance2_coloring_topology(topo, ne), want)


def _prototypes():
    """name -> number of parameters, parsed from the header's prototypes."""
    txt = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    out = {}
    for m in re.finditer(r"\b(ldg_[a-z0-9_]+)\s*\(([^;{]*?)\)\s*;", txt):
        args = m.group(2).strip()
        out[m.group(1)] = 0 if args in ("", "void") else args.count(",") + 1
    return out


def test_ctypes_signatures_match_header_arity():
    """Every argtypes list in _lib has exactly as many entries as the C
    prototype has parameters (a mismatch only shows up as a TypeError on the
    GPU box otherwise)."""
    protos = _prototypes()
    sigs = _lib._SIGS
    assert set(protos) >= set(sigs)
    for name, (argtypes, _) in sigs.items():
        assert len(argtypes) == protos[name], (name, len(argtypes), protos[name])
