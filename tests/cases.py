"""Parity cases shared by the golden generator and the tests.

Each case is built through a setup API module triple (model, mesh, master)
-- either the reference's ``ldgkit`` modules (golden generation, in the build
container only) or this package's ``model``/``meshgen``/``refelem`` (tests,
everywhere) -- so both sides see identical inputs.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).parent / "golden"

BOX_PERIODIC = {
    2: [(1, 2, (1.0, 0.0)), (3, 4, (0.0, 1.0))],
    3: [(1, 2, (1.0, 0.0, 0.0)), (3, 4, (0.0, 1.0, 0.0)), (5, 6, (0.0, 0.0, 1.0))],
}

# name -> spec
CASES = {
    "poisson3d_hex_p3": dict(model=("file", "poisson3d.model"), kind="hex",
                             counts=[2, 3, 2], p=3),
    "poisson3d_hex_p2": dict(model=("file", "poisson3d.model"), kind="hex",
                             counts=[3, 2, 2], p=2),
    "poisson2d_quad_p3": dict(model=("file", "poisson2d.model"), kind="quad",
                              counts=[3, 4], p=3),
    "poisson2d_quad_p1": dict(model=("file", "poisson2d.model"), kind="quad",
                              counts=[4, 3], p=1),
    "poisson2d_tri_p2": dict(model=("file", "poisson2d.model"), kind="tri",
                             counts=[3, 3], p=2),
    "poisson3d_tet_p2": dict(model=("file", "poisson3d.model"), kind="tet",
                             counts=[2, 2, 2], p=2),
    "convdiff3d_hex_periodic_p2": dict(
        model=("builtin", "convection_diffusion", 3, [0.7, -0.4, 1.1, 0.3]),
        kind="hex", counts=[3, 3, 3], p=2, periodic=3),
    "convdiff2d_quad_periodic_p3": dict(
        model=("builtin", "convection_diffusion", 2, [1.0, 0.5, 0.2]),
        kind="quad", counts=[3, 3], p=3, periodic=2),
    "convdiff2d_quad_dirichlet_p2": dict(
        model=("builtin", "convection_diffusion", 2, [0.8, -0.3, 0.5]),
        kind="quad", counts=[3, 2], p=2,
        bcs={t: ("dirichlet", ["x1*x2 + 0.5"]) for t in (1, 2, 3, 4)}),
    "poisson2d_quad_neumann_p2": dict(
        model=("builtin", "poisson", 2, None), kind="quad", counts=[3, 3], p=2,
        bcs={1: ("dirichlet", ["sin(x2)"]), 2: ("neumann", ["x2 - 0.25"]),
             3: ("dirichlet", ["0.5*x1"]), 4: ("neumann", ["cos(3*x1)"])}),
    "elasticity2d_quad_p2": dict(
        model=("builtin", "linear_elasticity", 2, [1.3, 0.8]), kind="quad",
        counts=[2, 3], p=2,
        bcs={t: ("dirichlet", ["0.1*x1", "-0.2*x2"]) for t in (1, 2, 3, 4)}),
    "poisson3d_hex_centered_p2": dict(
        model=("builtin", "poisson", 3, None), kind="hex", counts=[2, 2, 3], p=2,
        bcs={t: ("dirichlet", ["x1 + 2*x3"]) for t in range(1, 7)},
        numflux=dict(trace="centered", grad_trace="centered", tau=2.5)),
}

SOLVE_CASES = {
    # (case name, precond, solver flags)
    "poisson2d_quad_p3_n4_bj": dict(model=("file", "poisson2d.model"), kind="quad",
                                    counts=[4, 4], p=3, precond="block_jacobi"),
    "poisson2d_quad_p3_n4_id": dict(model=("file", "poisson2d.model"), kind="quad",
                                    counts=[4, 4], p=3, precond="identity"),
    "poisson3d_hex_p3_n2_bj": dict(model=("file", "poisson3d.model"), kind="hex",
                                   counts=[2, 2, 2], p=3, precond="block_jacobi"),
}

# acceptance solver flags (test_acceptance.py:69-81)
ACCEPT_FLAGS = dict(abs_tol=1e-11, rel_tol=3e-8, forcing=1e-8, restart=250,
                    gmres_max_iter=6000)


def build_case(spec, model_mod, mesh_mod, master_mod):
    """Return (model, mesh, topo, master) built with the given API modules."""
    src = spec["model"]
    if src[0] == "file":
        model = model_mod.load_model(str(GOLDEN / src[1]))
    else:
        _, name, nd, mu = src
        model = model_mod.builtin_model(name, nd=nd, mu=mu)
    if "bcs" in spec:
        model.bcs = {t: model_mod.BoundaryCondition(type=ty, data=list(d))
                     for t, (ty, d) in spec["bcs"].items()}
    if "init" in spec:
        model.init = {"u1": spec["init"]}
        model._plans = {}
    if "numflux" in spec:
        for k, v in spec["numflux"].items():
            setattr(model.numflux, k, v)
    kind = spec["kind"]
    nd = {"quad": 2, "tri": 2, "hex": 3, "tet": 3}[kind]
    mesh = mesh_mod.generate_structured([(0.0, 1.0)] * nd, spec["counts"], kind)
    per = BOX_PERIODIC[spec["periodic"]] if spec.get("periodic") else None
    if per is None and not model.bcs and spec.get("periodic") is None:
        pass
    topo = mesh_mod.build_face_topology(mesh, per)
    master = master_mod.build_master(kind, spec["p"])
    return model, mesh, topo, master


def seeded_state(ne, nb, ncu, seed):
    return np.random.default_rng(seed).normal(size=(ne, nb, ncu))


def b200_setup():
    from paper_2205_07824_b200 import meshgen, model, refelem
    return model, meshgen, refelem


# transient (DIRK) cases: reference advance_step (timeint.py:168-207)
TRANSIENT_CASES = {
    "convdiff2d_quad_p3_dirk22": dict(
        model=("builtin", "convection_diffusion", 2, [1.0, 0.5, 0.05]), kind="quad",
        counts=[6, 6], p=3, periodic=2, init="sin(2*pi*x1)*sin(2*pi*x2)",
        stages=2, order=2, dt=0.02, steps=3, precond="mass"),
    "convdiff3d_hex_p2_dirk11": dict(
        model=("builtin", "convection_diffusion", 3, [0.6, -0.3, 0.4, 0.05]), kind="hex",
        counts=[4, 4, 4], p=2, periodic=3, init="cos(2*pi*x1)*sin(2*pi*x3)",
        stages=1, order=1, dt=0.01, steps=2, precond="mass"),
}

TRANSIENT_FLAGS = dict(abs_tol=1e-10, rel_tol=1e-9, forcing=None, restart=60, gmres_max_iter=600)
