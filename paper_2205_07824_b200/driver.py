"""Callers of the hot path: steady closures, preconditioner wiring and the
steady solve (mirrors ``ldgkit/driver.py`` and ``ldgkit/timeint.py``).

``_steady_fns`` (driver.py:224-234), ``MassPreconditioner``
(driver.py:92-106), ``build_pde_block_jacobi`` (driver.py:119-125),
``make_preconditioner`` (driver.py:178-198, identity / mass / block_jacobi)
and ``solve_steady`` (timeint.py:210-241) keep the reference signatures;
vectors are device tensors end to end.
"""

from __future__ import annotations

import time

import numpy as np

from .solver import (NewtonOptions, build_block_jacobi, distance2_coloring,
                     element_neighbor_sets, newton_solve)


class DriverError(RuntimeError):
    pass


class TimeIntError(RuntimeError):
    pass


def _steady_fns(system):
    """Flat device closures R(u) and J(u) v at t = 0 (driver.py:224-234)."""
    shape = (system.n_elements, system.n_nodes, system.ncu)

    def residual(uflat):
        return system.residual_dev(uflat.reshape(shape), 0.0).reshape(-1)

    def tangent(uflat, v):
        return system.tangent_dev(v.reshape(shape)).reshape(-1)

    return residual, tangent


class MassPreconditioner:
    """Block inverse of the element mass operator (driver.py:92-106)."""

    def __init__(self, system):
        self.system = system

    def apply(self, r):
        s = self.system
        return s.mass_inv_dev(r.reshape(s.n_elements, s.n_nodes, s.ncu)).reshape(-1)


def build_pde_block_jacobi(system, residual_fn, tangent_fn, state_vec, jv_mode="tangent",
                           colors=None):
    """Exact per-element diagonal blocks via distance-2 coloured probing
    (driver.py:119-125)."""
    if jv_mode != "tangent":
        raise DriverError("the B200 block-Jacobi build probes the tangent operator")
    if colors is None:
        colors = distance2_coloring(element_neighbor_sets(system.topology, system.n_elements))
    return build_block_jacobi(tangent_fn, state_vec, system.n_elements,
                              system.n_nodes * system.ncu, colors)


def make_preconditioner(system, kind, residual_fn, tangent_fn, state_vec, steady=True,
                        jv_mode="tangent"):
    """driver.py:178-198 (identity, mass, block_jacobi)."""
    if kind == "auto":
        kind = "block_jacobi" if steady else "mass"
    if kind == "identity":
        return None, None
    if kind == "mass":
        return MassPreconditioner(system), None
    if kind == "block_jacobi":
        return build_pde_block_jacobi(system, residual_fn, tangent_fn, state_vec, jv_mode), None
    raise DriverError(f"unknown or unsupported preconditioner {kind!r}")


def solve_steady(system, state, newton_options=None, precond=None, callback=None):
    """Newton on R(u) = 0 (timeint.py:210-241).  Returns (state, stats)
    with state.u a device tensor."""
    from .system import SolverState
    if system.kind == "W":
        raise TimeIntError("steady solves do not apply to wave models")
    if not system.model.is_steady():
        raise TimeIntError("solve_steady requires a model with zero mass")
    opts = newton_options or NewtonOptions(forcing=1e-10)
    shape = (system.n_elements, system.n_nodes, system.ncu)
    t = state.t

    def residual(uflat):
        return system.residual_dev(uflat.reshape(shape), t).reshape(-1)

    def tangent(uflat, v):
        return system.tangent_dev(v.reshape(shape)).reshape(-1)

    import torch
    u0 = state.u if isinstance(state.u, torch.Tensor) else torch.as_tensor(
        np.ascontiguousarray(state.u, dtype=np.float64), device=system.device)
    x, stats = newton_solve(residual, u0.reshape(-1).cuda(), opts, precond=precond,
                            tangent_fn=tangent, callback=callback)
    return SolverState(u=x.reshape(shape), q=None, w=None, t=t), stats


def run_steady(system, precond="block_jacobi", abs_tol=1e-11, rel_tol=3e-8, forcing=1e-8,
               restart=250, gmres_max_iter=6000, max_iter=20, orth="mgs"):
    """Steady branch of run_simulation (driver.py:253-268) with the
    acceptance solver flags as defaults; returns (state, stats, timings)."""
    import torch
    t0 = time.perf_counter()
    state = system.interpolate_initial()
    res_fn, tan_fn = _steady_fns(system)
    u0 = torch.as_tensor(state.u, device=system.device).reshape(-1)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    M, cb = make_preconditioner(system, precond, res_fn, tan_fn, u0)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    opts = NewtonOptions(abs_tol=abs_tol, rel_tol=rel_tol, max_iter=max_iter, forcing=forcing,
                         gmres_restart=restart, gmres_max_iter=gmres_max_iter,
                         jv_mode="tangent", orth=orth)
    out, stats = solve_steady(system, state, opts, precond=M, callback=cb)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    if not stats.converged:
        raise DriverError(f"steady Newton solve did not converge "
                          f"(residual {stats.final_residual:.3e})")
    return out, stats, {"init_s": t1 - t0, "precond_build_s": t2 - t1, "solve_s": t3 - t2}
