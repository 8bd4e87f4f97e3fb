"""Generate golden vectors from the UNMODIFIED reference package.

Run in the build container (where the reference is mounted read-only):

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/gen_golden.py

Writes ``tests/golden/<case>.npz`` with the reference's topology arrays,
switch bits, residual R(u), tangent J(u)du, mixed gradient q(u) and
homogeneous dq(du) for each case in ``tests/cases.py``, plus Newton-GMRES
histories for the solve cases.  The reference never runs on the GPU box;
these committed files are what pins the oracle there.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, str(HERE.parent))

from ldgkit import master as R_master  # noqa: E402
from ldgkit import mesh as R_mesh  # noqa: E402
from ldgkit import model as R_model  # noqa: E402
from ldgkit.disc import LdgSystem, SolverState  # noqa: E402
from ldgkit.driver import _steady_fns, build_pde_block_jacobi  # noqa: E402
from ldgkit.solver import NewtonOptions  # noqa: E402
from ldgkit.timeint import solve_steady  # noqa: E402

from cases import (ACCEPT_FLAGS, BJ_CASES, CASES, CURVED_CASES, MB_CASES, NL_CASES,  # noqa: E402
                   SOLVE_CASES, mesh_arrays,
                   TRANSIENT_CASES, TRANSIENT_FLAGS, build_case, case_state, seeded_state)


def topo_arrays(sys_):
    t = sys_.topology
    return dict(elem_l=t.elem_l, face_l=t.face_l, elem_r=t.elem_r, face_r=t.face_r,
                translation=t.translation, elem_b=t.elem_b, face_b=t.face_b,
                tag_b=t.tag_b, n_true_interior=np.array(t.n_true_interior),
                switch=sys_.fi_switch, connectivity=sys_.mesh.connectivity)


def gen_case(name, spec):
    model, mesh, topo, master = build_case(spec, R_model, R_mesh, R_master)
    s = LdgSystem(model, mesh, topo, master)
    ne, nb, ncu = s.n_elements, s.n_nodes, s.ncu
    u = seeded_state(ne, nb, ncu, 1)
    du = seeded_state(ne, nb, ncu, 0)
    st = SolverState(u=u, q=None, w=None, t=0.0)
    R = s.residual(st)[0]
    J = s.residual_tangent(st, du)[0]
    out = dict(u=u, du=du, R=R, Jdu=J, **topo_arrays(s))
    if s.kind == "D":
        out["q"] = s.compute_mixed(u, 0.0)
        out["dq"] = s.compute_mixed(du, 0.0, homogeneous=True)
    out["node_x"] = s.disc.node_x
    out["fi_h"] = s.disc.fi_h
    out["mass_inv0"] = s.disc.mass_inv[0]
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, ne * nb * ncu, "dofs", float(np.abs(R).max()), float(np.abs(J).max()))


def gen_nl_case(name, spec):
    """Nonlinear / kind C operator goldens: R(u), J(u)du, compute_mixed,
    mass_apply and mass_tangent_extra at a physical base state."""
    model, mesh, topo, master = build_case(spec, R_model, R_mesh, R_master)
    s = LdgSystem(model, mesh, topo, master)
    ne, nb, ncu = s.n_elements, s.n_nodes, s.ncu
    u = case_state(spec, ne, nb, ncu, 1)
    du = seeded_state(ne, nb, ncu, 0)
    y = seeded_state(ne, nb, ncu, 2)
    st = SolverState(u=u, q=None, w=None, t=0.3)
    out = dict(u=u, du=du, y=y, t=np.array(0.3), R=s.residual(st)[0],
               Jdu=s.residual_tangent(st, du)[0], M=s.mass_apply(st, y)[0],
               **topo_arrays(s))
    ex = s.mass_tangent_extra(st, y, du)
    if ex is not None:
        out["Mx"] = ex
    if s.kind == "D":
        out["q"] = s.compute_mixed(u, 0.3)
        out["dq"] = s.compute_mixed(du, 0.3, homogeneous=True)
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, ne * nb * ncu, "dofs", float(np.abs(out["R"]).max()),
          float(np.abs(out["Jdu"]).max()))


def mb_states(s, spec):
    """Seeded packed-block states (u, q for kind W, w) and directions."""
    ne, nb = s.n_elements, s.n_nodes
    u = case_state(spec, ne, nb, s.ncu, 1)
    du = seeded_state(ne, nb, s.ncu, 0)
    q = dq = w = dw = None
    if s.kind == "W":
        q = np.random.default_rng(11).normal(size=(ne, nb, s.ncu, s.nd))
        dq = np.random.default_rng(12).normal(size=(ne, nb, s.ncu, s.nd))
    if s.nw > 0:
        w = 0.5 * np.random.default_rng(13).normal(size=(ne, nb, s.nw))
        dw = np.random.default_rng(14).normal(size=(ne, nb, s.nw))
    return u, q, w, du, dq, dw


def gen_mb_case(name, spec):
    """Packed multi-block operator goldens (kind W / ODE blocks)."""
    model, mesh, topo, master = build_case(spec, R_model, R_mesh, R_master)
    s = LdgSystem(model, mesh, topo, master)
    u, q, w, du, dq, dw = mb_states(s, spec)
    st = SolverState(u=u, q=q, w=w, t=0.2)
    out = dict(u=u, du=du, t=np.array(0.2), **topo_arrays(s))
    for k, v in (("q", q), ("dq", dq), ("w", w), ("dw", dw)):
        if v is not None:
            out[k] = v
    for tag, blocks in (("R", s.residual(st)), ("J", s.residual_tangent(st, du, dq, dw)),
                        ("M", s.mass_apply(st, du, dq, dw))):
        for bname, b in zip("uqw", blocks):
            if b is not None:
                out[f"{tag}{bname}"] = b
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, s.n_dofs, "dofs", sorted(k for k in out if k[0] in "RJM"))


def gen_solve(name, spec):
    model, mesh, topo, master = build_case(spec, R_model, R_mesh, R_master)
    s = LdgSystem(model, mesh, topo, master)
    st = s.interpolate_initial()
    f = ACCEPT_FLAGS
    opts = NewtonOptions(abs_tol=f["abs_tol"], rel_tol=f["rel_tol"], max_iter=20,
                         forcing=f["forcing"], gmres_restart=f["restart"],
                         gmres_max_iter=f["gmres_max_iter"],
                         jv_mode=spec.get("jv_mode", "tangent"))
    pre = cb = None
    if spec["precond"] in ("block_jacobi", "composite"):
        rf, tf = _steady_fns(s)
        pre = build_pde_block_jacobi(s, rf, tf, s.pack(st.u), spec.get("jv_mode", "tangent"))
        if spec["precond"] == "composite":
            # CompositeManager (driver.py:145-175) as make_preconditioner wires it
            from ldgkit.driver import CompositeManager
            pre = CompositeManager(s, pre, tf, rank=spec.get("rb_rank", 10), refresh=1)
            cb = pre.note_update
    out_state, stats = solve_steady(s, st, opts, precond=pre, callback=cb)
    extra = {}
    if "exact" in spec:
        from ldgkit.diagnostics import compute_l2_error
        eu, eq = spec["exact"]
        err = compute_l2_error(s, out_state, eu, eq)
        extra = dict(error_u=np.array(err.error_u))
        if err.error_q is not None:
            extra["error_q"] = np.array(err.error_q)
    np.savez_compressed(HERE / f"solve_{name}.npz", u=out_state.u,
                        newton_iters=np.array(stats.newton_iters),
                        gmres_iters=np.array(stats.gmres_iters),
                        residual_norms=np.array(stats.residual_norms), **extra)
    print("solve", name, stats.newton_iters, stats.gmres_iters, extra)


def gen_transient(name, spec):
    from ldgkit.driver import MassPreconditioner
    from ldgkit.timeint import advance_step, dirk_tableau
    model, mesh, topo, master = build_case(spec, R_model, R_mesh, R_master)
    s = LdgSystem(model, mesh, topo, master)
    st = s.interpolate_initial()
    f = TRANSIENT_FLAGS
    opts = NewtonOptions(abs_tol=f["abs_tol"], rel_tol=f["rel_tol"], max_iter=20,
                         forcing=f["forcing"], gmres_restart=f["restart"],
                         gmres_max_iter=f["gmres_max_iter"], jv_mode="tangent")
    tab = dirk_tableau(spec["stages"], spec["order"])
    extra = {}
    if spec["precond"] == "block_jacobi":
        # transient block-Jacobi: built once at t = 0 from the steady
        # closures (driver.py:270-274)
        rf, tf = _steady_fns(s)
        M = build_pde_block_jacobi(s, rf, tf, s.pack(st.u), "tangent")
    else:
        M = MassPreconditioner(s)
    newton, gm, per_newton, per_stage = [], [], [], []
    u0 = st.u.copy()
    for _ in range(spec["steps"]):
        st, stats = advance_step(s, st, spec["dt"], tab, opts, precond=M)
        newton.append(stats.newton_iters)
        gm.append(stats.gmres_iters)
        for ss in stats.stage_stats:            # GMRES count of every Newton step, by stage
            per_stage.append(len(ss.gmres_iters))
            per_newton.extend(int(x) for x in ss.gmres_iters)
    extra.update(gmres_newton=np.array(per_newton, dtype=np.int64),
                 gmres_stage_len=np.array(per_stage, dtype=np.int64))
    if st.q is not None or st.w is not None:
        extra.update({k: v for k, v in (("q", st.q), ("w", st.w)) if v is not None})
    if spec.get("bj_apply"):
        # block-Jacobi of the steady closures at the initial state, applied
        # to a seeded vector (solver.py:291-346, driver.py:109-142)
        s0 = s.interpolate_initial()
        rf, tf = _steady_fns(s)
        bj = build_pde_block_jacobi(s, rf, tf, s.pack(s0.u), "tangent")
        r = np.random.default_rng(9).normal(size=s.n_dofs)
        extra.update(bj_r=r, bj_z=bj.apply(r))
    np.savez_compressed(HERE / f"transient_{name}.npz", u0=u0, u=st.u, t=np.array(st.t),
                        newton=np.array(newton), gmres=np.array(gm), **extra)
    print("transient", name, newton, gm, float(np.abs(st.u).max()))


def gen_curved(name, spec):
    """Curved / non-affine meshes (disc.py:91-180 per-point geometry): the
    mesh arrays, R at the free stream, R / J du / M y at a perturbed state."""
    model, mesh, topo, master = build_case(spec, R_model, R_mesh, R_master)
    s = LdgSystem(model, mesh, topo, master)
    ne, nb, ncu = s.n_elements, s.n_nodes, s.ncu
    u = case_state(spec, ne, nb, ncu, 1)
    du = seeded_state(ne, nb, ncu, 0)
    y = seeded_state(ne, nb, ncu, 2)
    st = SolverState(u=u, q=None, w=None, t=0.0)
    out = dict(u=u, du=du, y=y, R=s.residual(st)[0], Jdu=s.residual_tangent(st, du)[0],
               M=s.mass_apply(st, y)[0], **mesh_arrays(mesh), **topo_arrays(s))
    if "free" in spec:
        uf = np.broadcast_to(np.asarray(spec["free"], dtype=float), (ne, nb, ncu)).copy()
        out.update(u_free=uf, R_free=s.residual(SolverState(u=uf, q=None, w=None, t=0.0))[0])
    if s.kind == "D":
        out.update(q=s.compute_mixed(u, 0.0), dq=s.compute_mixed(du, 0.0, homogeneous=True))
    np.savez_compressed(HERE / spec["mesh_file"], **out)
    print("curved", name, ne * nb * ncu, "free-stream |R|",
          float(np.abs(out["R_free"]).max()) if "R_free" in out else None)


def gen_bj(name, spec):
    """The reference's block-Jacobi of the steady closures at the initial
    state (driver.py:119-142, solver.py:303-346) applied to a seeded vector."""
    model, mesh, topo, master = build_case(spec, R_model, R_mesh, R_master)
    s = LdgSystem(model, mesh, topo, master)
    s0 = s.interpolate_initial()
    rf, tf = _steady_fns(s)
    bj = build_pde_block_jacobi(s, rf, tf, s.pack(s0.u), "tangent")
    r = np.random.default_rng(9).normal(size=s.n_dofs)
    np.savez_compressed(HERE / f"{name}.npz", bj_r=r, bj_z=bj.apply(r))
    print("bj", name, s.n_dofs)


if __name__ == "__main__":
    if "--curved-only" in sys.argv:
        for n, sp in CURVED_CASES.items():
            gen_curved(n, sp)
        sys.exit(0)
    if "--bj-only" in sys.argv:
        for n, sp in BJ_CASES.items():
            gen_bj(n, sp)
        sys.exit(0)
    if "--nl-only" in sys.argv:
        for n, sp in NL_CASES.items():
            gen_nl_case(n, sp)
        sys.exit(0)
    if "--mb-only" in sys.argv:
        for n, sp in MB_CASES.items():
            gen_mb_case(n, sp)
        sys.exit(0)
    if "--transient-only" in sys.argv:
        for n, sp in TRANSIENT_CASES.items():
            if len(sys.argv) > 2 and n not in sys.argv:
                continue
            gen_transient(n, sp)
        sys.exit(0)
    if "--solve-only" in sys.argv:
        for n, sp in SOLVE_CASES.items():
            if len(sys.argv) > 2 and n not in sys.argv:
                continue
            gen_solve(n, sp)
        sys.exit(0)
    for n, sp in CASES.items():
        gen_case(n, sp)
    for n, sp in NL_CASES.items():
        gen_nl_case(n, sp)
    for n, sp in MB_CASES.items():
        gen_mb_case(n, sp)
    for n, sp in SOLVE_CASES.items():
        gen_solve(n, sp)
    for n, sp in TRANSIENT_CASES.items():
        gen_transient(n, sp)
    for n, sp in BJ_CASES.items():
        gen_bj(n, sp)
    for n, sp in CURVED_CASES.items():
        gen_curved(n, sp)
