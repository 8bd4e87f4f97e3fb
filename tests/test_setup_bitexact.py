"""Setup layer (reference element, mesh, face topology) is bit-exact with
the reference: against committed golden arrays everywhere, and against the
live reference package when it is importable (build container)."""

import sys

import numpy as np
import pytest

from cases import CASES, GOLDEN, b200_setup, build_case
from conftest import REFERENCE_SRC, reference_available

TOPO = ("elem_l", "face_l", "elem_r", "face_r", "translation", "elem_b",
        "face_b", "tag_b")


@pytest.mark.parametrize("name", sorted(CASES))
def test_topology_matches_golden(name):
    g = np.load(GOLDEN / f"{name}.npz")
    model, mesh, topo, master = build_case(CASES[name], *b200_setup())
    assert np.array_equal(mesh.connectivity, g["connectivity"])
    for k in TOPO:
        assert np.array_equal(getattr(topo, k), g[k]), k
    assert topo.n_true_interior == int(g["n_true_interior"])


needs_ref = pytest.mark.skipif(not reference_available(),
                               reason="reference package not mounted")


@needs_ref
@pytest.mark.parametrize("kind,p", [(k, p) for k in ("line", "tri", "quad", "tet", "hex")
                                    for p in range(1, 9)])
def test_master_bitexact_vs_reference(kind, p):
    sys.path.insert(0, REFERENCE_SRC)
    from ldgkit import master as RM
    from paper_2205_07824_b200 import refelem
    pairs = [(RM.build_master(kind, p), refelem.build_master(kind, p))]
    if p <= 3:
        pairs.append((RM.build_geom_master(kind, p), refelem.build_geom_master(kind, p)))
    for a, b in pairs:
        for nm in ("nodes", "quad_pts", "quad_wts", "phi", "dphi", "vandermonde",
                   "vandermonde_inv", "nodes1d", "phi1d", "dphi1d"):
            x, y = getattr(a, nm), getattr(b, nm)
            assert (x is None and y is None) or np.array_equal(x, y), nm
        assert a.n_faces == b.n_faces and a.quad_degree == b.quad_degree
        for fa, fb in zip(a.faces, b.faces):
            for nm in ("sigma", "weights", "xi", "phi"):
                assert np.array_equal(getattr(fa, nm), getattr(fb, nm)), nm
        pts = a.quad_pts[::2]
        assert np.array_equal(a.eval_basis_grad(pts), b.eval_basis_grad(pts))


@needs_ref
@pytest.mark.parametrize("kind,counts,per", [
    ("hex", [3, 2, 4], None), ("tet", [2, 3, 2], None), ("quad", [5, 3], None),
    ("tri", [4, 4], None), ("hex", [3, 3, 3], 3), ("tet", [2, 2, 2], 3),
    ("tri", [3, 4], 2), ("quad", [4, 2], 2)])
def test_mesh_topology_bitexact_vs_reference(kind, counts, per):
    sys.path.insert(0, REFERENCE_SRC)
    from ldgkit import mesh as RM
    from cases import BOX_PERIODIC
    from paper_2205_07824_b200 import meshgen
    nd = len(counts)
    spec = BOX_PERIODIC[per] if per else None
    for pg in (1, 2):
        m1 = RM.generate_structured([(0, 1)] * nd, counts, kind, p_geom=pg)
        m2 = meshgen.generate_structured([(0, 1)] * nd, counts, kind, p_geom=pg)
        for nm in ("vertices", "connectivity", "ho_nodes", "boundary_faces"):
            assert np.array_equal(getattr(m1, nm), getattr(m2, nm)), nm
        t1 = RM.build_face_topology(m1, spec)
        t2 = meshgen.build_face_topology(m2, spec)
        for k in TOPO:
            assert np.array_equal(getattr(t1, k), getattr(t2, k)), k
        assert np.array_equal(np.array(t1.perm), np.array(t2.perm))


def test_simplex_face_orientation_from_vertex_ids_matches_geometry():
    """DenseTables._orient_fast (shared vertex ids, geometry only for
    periodic faces) == the geometric point matching on every face."""
    from paper_2205_07824_b200 import meshgen, model, refelem
    from paper_2205_07824_b200.tables import DenseTables
    root = GOLDEN
    for kind, counts, per, p in (("tet", [5, 4, 3], None, 2), ("tri", [6, 5], None, 3),
                                 ("tri", [4, 4], [(1, 2, (1.0, 0.0)), (3, 4, (0.0, 1.0))], 3),
                                 ("tet", [3, 3, 3], [(1, 2, (1.0, 0.0, 0.0))], 2)):
        nd = len(counts)
        m = model.load_model(str(root / ("poisson3d.model" if nd == 3 else "poisson2d.model")))
        mesh = meshgen.generate_structured([(0.0, 1.0)] * nd, counts, kind)
        topo = meshgen.build_face_topology(mesh, per)
        T = DenseTables(m, mesh, topo, refelem.build_master(kind, p))
        el, fl, er, fr = (np.asarray(a, dtype=np.int64) for a in
                          (topo.elem_l, topo.face_l, topo.elem_r, topo.face_r))
        tr = np.asarray(topo.translation, dtype=float)
        if tr.shape[0] != el.size:
            tr = np.zeros((el.size, nd))
        assert np.array_equal(T._orient(el, fl, er, fr, tr), T._orient_fast(el, fl, er, fr, tr))
        assert np.array_equal(T._orient(er, fr, el, fl, -tr), T._orient_fast(er, fr, el, fl, -tr))
