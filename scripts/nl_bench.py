"""Throughput of the generated-kernel path (nonlinear.py) on the BASELINE
nonlinear configs:

  config 4 shape: 3D compressible Navier-Stokes (tests/golden/ns3d.model),
                  periodic hex p=3, n^3 elements (n=32: 10.5M DOFs)
  config 2 shape: 2D Euler isentropic vortex, periodic quad p=4 on [0,10]^2

    python scripts/nl_bench.py [--ns-n 32] [--euler-n 256] [--reps 20]

Times residual R(u) and tangent J(u)du (base mixed gradient cached, as in
Newton-GMRES) with CUDA events on the launching stream, L2 flushed between
reps; prints one JSON line with GDOF/s, per-kernel times and the achieved
bandwidth against the SURVEY 8(d) byte counts (kind D nonlinear tangent
104 B/DOF in 3D; kind C tangent 24 B/DOF)."""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def timed(fn, reps, flush):
    import torch
    st = torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def run(name, spec, reps, peak):
    import torch
    from cases import build_case, b200_setup, case_state
    from paper_2205_07824_b200.system import LdgSystem
    model, mesh, topo, master = build_case(spec, *b200_setup())
    s = LdgSystem(model, mesh, topo, master)
    shape = (s.n_elements, s.n_nodes, s.ncu)
    u = torch.as_tensor(case_state(spec, *shape, 1), device="cuda")
    du = torch.as_tensor(np.random.default_rng(0).normal(size=shape), device="cuda")
    out = torch.empty_like(u)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    q = s.base_mixed(u, 0.0)
    nl = s.nl
    dq = nl.mixed(du, 0.0, homogeneous=True) if q is not None else None
    for _ in range(3):
        nl.tangent(u, du, 0.0, q=q, out=out)
        nl.residual(u, 0.0, q=q, out=out)
    torch.cuda.synchronize()
    r = {"dofs": s.n_dofs, "kind": model.kind, "ncu": s.ncu, "p": master.p,
         "elements": s.n_elements}
    r["residual_ms"] = timed(lambda: nl.residual(u, 0.0, q=q, out=out), reps, flush)
    # GMRES matvec: the base state's point values come from the per-base
    # cache (built once per Newton step, timed separately); the uncached
    # tangent (the base interpolated every call) beside it
    r["tangent_ms"] = timed(lambda: nl.tangent(u, du, 0.0, q=q, out=out), reps, flush)
    r["tangent_cached_ms"] = timed(lambda: nl.tangent(u, du, 0.0, q=q, out=out, cached=True),
                                   reps, flush)
    r["tangent_uncached_ms"] = timed(lambda: nl.tangent(u, du, 0.0, q=q, out=out, cached=False),
                                     reps, flush)

    def rebuild():
        nl._bkey = None
        nl.base_cache(u, 0.0, q)
    r["base_cache_ms"] = timed(rebuild, reps, flush)
    if q is not None:
        r["mixed_ms"] = timed(lambda: nl.mixed(du, 0.0, True, out=dq), reps, flush)
        P = nl._params(0.0, u=u, q=q, du=du, dq=dq, out=out, gq=nl.gq(0.0))
        r["tangent_kernel_ms"] = timed(
            lambda: nl._launch("nl_tangent", s.n_elements, nl.shape["NT"], P), reps, flush)
        nd = mesh.nd
        bpd = 8 * (4 + 3 * nd)           # kind D nonlinear tangent
    else:
        r["tangent_kernel_ms"] = r["tangent_ms"]
        bpd = 24                          # kind C tangent: du, base u, dR
    r["tangent_gdofs"] = s.n_dofs / r["tangent_ms"] / 1e6
    r["tangent_uncached_gdofs"] = s.n_dofs / r["tangent_uncached_ms"] / 1e6
    r["residual_gdofs"] = s.n_dofs / r["residual_ms"] / 1e6
    r["tangent_bytes_per_dof"] = bpd
    r["tangent_achieved_gbs"] = bpd * s.n_dofs / r["tangent_ms"] / 1e6
    r["tangent_frac_hbm"] = r["tangent_achieved_gbs"] / peak
    r["attrs"] = {k: nl.kernel_attrs(k) for k in ("nl_residual", "nl_tangent", "nl_tangent_cached",
                                                   "nl_mixed")}
    return name, r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns-n", type=int, default=32)
    ap.add_argument("--euler-n", type=int, default=256)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    from cases import NL_CASES, TRANSIENT_CASES
    try:
        peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    except Exception:
        peak = 6553.0
    out = {}
    ns = dict(TRANSIENT_CASES["ns3d_tgv_hex_p2_dirk11"], counts=[a.ns_n] * 3, p=3,
              state=([1.0, 0.2, -0.1, 0.15, 25.0], 0.05))
    eu = dict(TRANSIENT_CASES["euler2d_vortex_quad_p3_dirk22"], counts=[a.euler_n] * 2, p=4,
              state=([1.0, 0.2, -0.1, 2.5], 0.05))
    for name, spec in (("config4_ns3d_hex_p3", ns), ("config2_euler2d_quad_p4", eu)):
        k, v = run(name, spec, a.reps, peak)
        out[k] = v
    del NL_CASES
    print(json.dumps(out))



def run_transient(spec, steps, dt, precond="mass", flags=None):
    """Wall time per implicit DIRK step (device Newton-GMRES, reference
    transient solver flags), with Newton / GMRES counts."""
    import time
    import torch
    from cases import TRANSIENT_FLAGS, build_case, b200_setup
    from paper_2205_07824_b200.driver import MassPreconditioner, advance_step, dirk_tableau
    from paper_2205_07824_b200.solver import NewtonOptions
    from paper_2205_07824_b200.system import LdgSystem
    f = dict(TRANSIENT_FLAGS, **(flags or {}))
    s = LdgSystem(*build_case(spec, *b200_setup()))
    st = s.interpolate_initial()
    opts = NewtonOptions(abs_tol=f["abs_tol"], rel_tol=f["rel_tol"], max_iter=20,
                         forcing=f["forcing"], gmres_restart=f["restart"],
                         gmres_max_iter=f["gmres_max_iter"], jv_mode="tangent",
                         orth=f.get("orth", "cgs2"))
    tab = dirk_tableau(spec["stages"], spec["order"])
    build_s = 0.0
    if precond == "block_jacobi":
        # the reference's transient block-Jacobi: built once from the steady
        # closures at the initial state (driver.py:270-274)
        from paper_2205_07824_b200.driver import _steady_fns, build_pde_block_jacobi
        t0 = time.perf_counter()
        rf, tf = _steady_fns(s)
        M = build_pde_block_jacobi(s, rf, tf, torch.as_tensor(st.u, device=s.device).reshape(-1))
        torch.cuda.synchronize()
        build_s = time.perf_counter() - t0
    else:
        M = MassPreconditioner(s)
    from paper_2205_07824_b200.driver import TimeIntError
    try:
        st, _ = advance_step(s, st, dt, tab, opts, precond=M)   # warm-up (JIT, caches)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        newton, gm = [], []
        for _ in range(steps):
            st, stats = advance_step(s, st, dt, tab, opts, precond=M)
            newton.append(stats.newton_iters)
            gm.append(stats.gmres_iters)
        torch.cuda.synchronize()
    except TimeIntError as exc:
        return {"dofs": s.n_dofs, "dt": dt, "failed": str(exc)}
    per = (time.perf_counter() - t0) / steps
    return {"dofs": s.n_dofs, "dt": dt, "steps": steps, "s_per_step": per,
            "newton_per_step": newton, "gmres_per_step": gm, "precond": precond,
            "precond_build_s": build_s,
            "max_abs_u": float(torch.max(torch.abs(st.u)).item())}


def cpu_oracle_tangent(spec, reps=2):
    """The oracle (reference numpy path) tangent on a small sample of a
    config: GDOF/s on this host, 1 core."""
    import time
    from cases import build_case, b200_setup, case_state
    from oracle import make_oracle
    model, mesh, topo, master = build_case(spec, *b200_setup())
    o = make_oracle(model, mesh, topo, master)
    ne, nb, ncu = mesh.connectivity.shape[0], master.n_nodes, model.ncu
    u = case_state(spec, ne, nb, ncu, 1)
    du = np.random.default_rng(0).normal(size=u.shape)
    o.residual_tangent(u, du)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        o.residual_tangent(u, du)
        ts.append(time.perf_counter() - t0)
    return {"dofs": ne * nb * ncu, "gdofs": ne * nb * ncu / float(np.median(ts)) / 1e9,
            "cores": 1, "kind": "port"}


if __name__ == "__main__":
    main()
