"""Host table builder + the tensor kernels' algebra, emulated in numpy on
CPU, against the reference golden vectors (no GPU needed)."""

import numpy as np
import pytest

import tensor_emulation as emu
from cases import CASES, GOLDEN, b200_setup, build_case
from paper_2205_07824_b200.tables import DiscError, TensorTables

TENSOR = sorted(n for n, s in CASES.items() if s["kind"] in ("quad", "hex"))


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name", TENSOR)
def test_tensor_algebra_matches_reference(name):
    g = np.load(GOLDEN / f"{name}.npz")
    tab = TensorTables(*build_case(CASES[name], *b200_setup()))
    assert np.array_equal(tab.switch, g["switch"])
    gp, bs = tab.boundary_projection(0.0), tab.source_load(0.0)
    q = emu.mixed(tab, g["u"], gp)
    dq = emu.mixed(tab, g["du"], None)
    assert rel(q, g["q"]) < 1e-13
    assert rel(dq, g["dq"]) < 1e-13
    assert rel(emu.flux(tab, g["u"], q, False, gp, bs), g["R"]) < 1e-13
    assert rel(emu.flux(tab, g["du"], dq, True), g["Jdu"]) < 1e-13
    assert rel(tab.fi_h, g["fi_h"]) < 1e-13
    # the fused two-pass split (ldg_fused.cu) reproduces the same operator
    assert rel(emu.fused(tab, g["u"], False, gp, bs), g["R"]) < 1e-13
    assert rel(emu.fused(tab, g["du"], True), g["Jdu"]) < 1e-13


@pytest.mark.parametrize("name", ["poisson2d_tri_p2", "poisson3d_tet_p2"])
def test_simplex_rejected_loudly(name):
    with pytest.raises(DiscError):
        TensorTables(*build_case(CASES[name], *b200_setup()))


def test_nonlinear_flux_rejected():
    from paper_2205_07824_b200 import model as M
    m = M.builtin_model("poisson", nd=2)
    m.flux = ["q1_1*u1", "q1_2"]
    m._plans = {}
    m.bcs = {t: M.BoundaryCondition("dirichlet", ["0"]) for t in (1, 2, 3, 4)}
    _, mesh, topo, master = build_case(CASES["poisson2d_quad_p1"], *b200_setup())
    with pytest.raises(DiscError):
        TensorTables(m, mesh, topo, master)


def test_node_maps_config3_structure():
    """Structured hex meshes need exactly 6 neighbour maps (one per face)."""
    from paper_2205_07824_b200 import meshgen, model, refelem
    m = model.builtin_model("poisson", nd=3)
    m.bcs = {t: model.BoundaryCondition("dirichlet", ["0"]) for t in range(1, 7)}
    mesh = meshgen.generate_structured([(0, 1)] * 3, [6, 5, 4], "hex")
    tab = TensorTables(m, mesh, meshgen.build_face_topology(mesh), refelem.build_master("hex", 3))
    assert tab.nmap.shape == (6, 16)
    assert tab.switch.all()


@pytest.mark.parametrize("name", ["poisson2d_tri_p2", "poisson3d_tet_p2"])
def test_dense_algebra_matches_reference(name):
    import dense_emulation as de
    from paper_2205_07824_b200.tables import DenseTables
    g = np.load(GOLDEN / f"{name}.npz")
    t = DenseTables(*build_case(CASES[name], *b200_setup()))
    assert np.array_equal(t.switch, g["switch"])
    gv, bs = t.boundary_values(0.0), t.source_load(0.0)
    q, dq = de.mixed(t, g["u"], gv), de.mixed(t, g["du"])
    assert rel(q, g["q"]) < 1e-13 and rel(dq, g["dq"]) < 1e-13
    assert rel(de.flux(t, g["u"], q, False, gv, bs), g["R"]) < 1e-13
    assert rel(de.flux(t, g["du"], dq, True), g["Jdu"]) < 1e-13


def _ldgkit_setup():
    import sys
    from conftest import REFERENCE_SRC
    sys.path.insert(0, REFERENCE_SRC)
    from ldgkit import master as RMa
    from ldgkit import mesh as RMe
    from ldgkit import model as RMo
    return RMo, RMe, RMa


@pytest.mark.skipif(not __import__("conftest").reference_available(),
                    reason="reference package not mounted")
@pytest.mark.parametrize("name", ["poisson3d_hex_p3", "convdiff3d_hex_periodic_p2",
                                  "poisson2d_tri_p2", "poisson3d_tet_p2"])
def test_dropin_tables_from_ldgkit_objects(name):
    """The drop-in claim: the device tables built from ldgkit's OWN setup
    objects (PdeModel, Mesh, FaceTopology, MasterElement; disc.py:265) give
    the reference operator, i.e. the B200 LdgSystem accepts exactly what a
    reference caller passes."""
    from paper_2205_07824_b200.tables import DenseTables
    g = np.load(GOLDEN / f"{name}.npz")
    parts = build_case(CASES[name], *_ldgkit_setup())
    if CASES[name]["kind"] in ("quad", "hex"):
        tab = TensorTables(*parts)
        assert np.array_equal(tab.switch, g["switch"])
        gp, bs = tab.boundary_projection(0.0), tab.source_load(0.0)
        assert rel(emu.fused(tab, g["u"], False, gp, bs), g["R"]) < 1e-13
        assert rel(emu.fused(tab, g["du"], True), g["Jdu"]) < 1e-13
    else:
        import dense_emulation as de
        t = DenseTables(*parts)
        assert np.array_equal(t.switch, g["switch"])
        gv, bs = t.boundary_values(0.0), t.source_load(0.0)
        q = de.mixed(t, g["u"], gv)
        assert rel(de.flux(t, g["u"], q, False, gv, bs), g["R"]) < 1e-13
        assert rel(de.flux(t, g["du"], de.mixed(t, g["du"]), True), g["Jdu"]) < 1e-13


@pytest.mark.skipif(not __import__("conftest").reference_available(),
                    reason="reference package not mounted")
@pytest.mark.parametrize("name", ["euler2d_quad_periodic_p3", "ns3d_hex_periodic_p2"])
def test_dropin_nl_tables_from_ldgkit_objects(name):
    """Generated-kernel tables (NlTables) accept ldgkit's objects and agree
    with the ones built from this package's setup restatement."""
    from cases import NL_CASES
    from paper_2205_07824_b200.nonlinear import NlTables
    a = NlTables(*build_case(NL_CASES[name], *_ldgkit_setup()))
    b = NlTables(*build_case(NL_CASES[name], *b200_setup()))
    g = np.load(GOLDEN / f"{name}.npz")
    assert np.array_equal(a.switch, g["switch"])
    for k in ("geo", "xmap", "fgeo", "fnbr", "finfo"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
