"""Newton-GMRES time-to-solution for 3D Poisson hex p=3 (config 3) on the
B200 path, with the reference's acceptance solver flags.

    python scripts/solve_bench.py --n 54 --orth cgs2 [--cpu-n 4]

Prints one JSON line: precond build / solve seconds, Newton and GMRES
counts, L2 error against the manufactured solution; with --cpu-n the
oracle (reference numpy path) solves the n=cpu_n case for comparison.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def build(n, p=3):
    from paper_2205_07824_b200 import meshgen, model, refelem
    m = model.load_model(str(ROOT / "tests" / "golden" / "poisson3d.model"))
    mesh = meshgen.generate_structured([(0.0, 1.0)] * 3, [n] * 3, "hex")
    return m, mesh, meshgen.build_face_topology(mesh), refelem.build_master("hex", p)


def l2_error(system, u):
    """Relative L2 error vs sin(pi x) sin(pi y) sin(pi z) by quadrature
    (diagnostics.py:35-65)."""
    xq = system.disc.xq
    w = system.disc.wdetj
    uq = np.einsum("qa,ea->eq", system.master.phi, u.reshape(system.n_elements, -1))
    ex = np.sin(np.pi * xq[..., 0]) * np.sin(np.pi * xq[..., 1]) * np.sin(np.pi * xq[..., 2])
    return float(np.sqrt(np.sum(w * (uq - ex) ** 2) / np.sum(w * ex ** 2)))


def gpu_solve(n, orth, restart):
    import torch
    from paper_2205_07824_b200.driver import run_steady
    from paper_2205_07824_b200.system import LdgSystem
    t0 = time.perf_counter()
    s = LdgSystem(*build(n))
    setup = time.perf_counter() - t0
    st, stats, tm = run_steady(s, precond="block_jacobi", restart=restart, orth=orth)
    torch.cuda.synchronize()
    # a second solve on the same system: the Krylov workspace (20 GB at
    # restart 250) and the caching allocator are warm
    _, _, tm2 = run_steady(s, precond="block_jacobi", restart=restart, orth=orth)
    torch.cuda.synchronize()
    return {"n": n, "dofs": s.n_dofs, "orth": orth, "setup_s": setup, **tm,
            "warm_precond_build_s": tm2["precond_build_s"], "warm_solve_s": tm2["solve_s"],
            "newton": stats.newton_iters, "gmres": stats.total_gmres_iters,
            "final_residual": stats.final_residual,
            "error_u": l2_error(s, st.u.cpu().numpy())}


def cpu_solve(n):
    from oracle import make_oracle
    from oracle.solver_oracle import (block_jacobi_blocks, block_jacobi_factor,
                                      distance2_coloring, element_neighbors, newton_solve)
    m, mesh, topo, master = build(n)
    o = make_oracle(m, mesh, topo, master)
    ne, nb = mesh.connectivity.shape[0], master.n_nodes
    t0 = time.perf_counter()
    colors = distance2_coloring(element_neighbors(topo, ne))
    tan = lambda x, v: o.residual_tangent(x.reshape(ne, nb, 1), v.reshape(ne, nb, 1)).ravel()  # noqa: E731
    mats = block_jacobi_blocks(tan, np.zeros(ne * nb), ne, nb, colors)
    M = block_jacobi_factor(mats)
    t1 = time.perf_counter()
    res = lambda x: o.residual(x.reshape(ne, nb, 1)).ravel()  # noqa: E731
    x, st = newton_solve(res, tan, np.zeros(ne * nb), abs_tol=1e-11, rel_tol=3e-8,
                         forcing=1e-8, restart=250, gmres_max_iter=6000, precond=M)
    t2 = time.perf_counter()
    return {"n": n, "dofs": ne * nb, "precond_build_s": t1 - t0, "solve_s": t2 - t1,
            "newton": st["newton_iters"], "gmres": int(sum(st["gmres_iters"]))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=54)
    ap.add_argument("--orth", default="dcgs2")
    ap.add_argument("--restart", type=int, default=250)
    ap.add_argument("--cpu-n", type=int, default=0)
    a = ap.parse_args()
    out = {"gpu": gpu_solve(a.n, a.orth, a.restart)}
    if a.cpu_n:
        out["cpu_oracle"] = cpu_solve(a.cpu_n)
        out["gpu_same_n"] = gpu_solve(a.cpu_n, a.orth, a.restart)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
