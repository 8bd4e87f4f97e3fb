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

from .solver import (BlockJacobiPreconditioner, NewtonOptions, build_block_jacobi,
                     distance2_coloring, distance2_coloring_topology, element_neighbor_sets,
                     newton_solve)


class DriverError(RuntimeError):
    pass


class TimeIntError(RuntimeError):
    pass


def _steady_fns(system):
    """Flat device closures R(u) and J(u) v at t = 0 (driver.py:224-234);
    packed (u | q | w) vectors for kind W / ODE systems."""
    if getattr(system, "multi_block", False):
        return (lambda Y: system.residual_packed_dev(Y, 0.0),
                lambda Y, V: system.tangent_packed_dev(V, Y, 0.0))
    shape = (system.n_elements, system.n_nodes, system.ncu)

    def residual(uflat):
        return system.residual_dev(uflat.reshape(shape), 0.0).reshape(-1)

    def tangent(uflat, v):
        return system.tangent_dev(v.reshape(shape), base=uflat.reshape(shape)).reshape(-1)

    tangent.steady_tangent_of = system     # lets the block-Jacobi build probe natively
    return residual, tangent


class MassPreconditioner:
    """Block inverse of the element mass operator (driver.py:92-106)."""

    def __init__(self, system):
        self.system = system

    def apply(self, r):
        s = self.system
        if getattr(s, "multi_block", False):
            return s.mass_inv_packed_dev(r)
        return s.mass_inv_dev(r.reshape(s.n_elements, s.n_nodes, s.ncu)).reshape(-1)


def elementwise_block_perm(system, device):
    """Per-element dof indices across the packed (u, q, w) blocks
    (driver.py:128-142, ``_elementwise_blocks``) as one int64 device vector:
    perm[e*bs + j] = packed index of row j of element e's block."""
    import torch
    ne, nb = system.n_elements, system.n_nodes
    sizes = [nb * system.ncu]
    if system.kind == "W":
        sizes.append(nb * system.ncu * system.nd)
    if getattr(system, "nw", 0) > 0:
        sizes.append(nb * system.nw)
    offsets = np.cumsum([0] + [ne * s for s in sizes])
    e = np.arange(ne, dtype=np.int64)[:, None]
    cols = [off + e * s + np.arange(s, dtype=np.int64)[None, :]
            for off, s in zip(offsets[:-1], sizes)]
    return torch.as_tensor(np.concatenate(cols, axis=1).reshape(-1), device=device), sum(sizes)


def build_pde_block_jacobi(system, residual_fn, tangent_fn, state_vec, jv_mode="tangent",
                           colors=None, invert="auto", share=True, scratch=None):
    """Exact per-element diagonal blocks via distance-2 coloured probing
    (driver.py:119-142), through the tangent or by finite differences
    (``jv_mode``), across the packed blocks of kind-W / ODE systems."""
    if colors is None:
        colors = distance2_coloring_topology(system.topology, system.n_elements)
    from .system import LdgSystem
    import torch
    x = state_vec if isinstance(state_vec, torch.Tensor) else \
        torch.as_tensor(np.asarray(state_vec, dtype=np.float64), device=system.device)
    if getattr(system, "multi_block", False):
        perm, bs = elementwise_block_perm(system, x.device)
        return build_block_jacobi(tangent_fn, x, system.n_elements, bs, colors, perm=perm,
                                  mode=jv_mode, residual_fn=residual_fn, invert=invert,
                                  share=share)
    native = None
    if (jv_mode == "tangent" and type(system) is LdgSystem and system.nl is None
            and getattr(system, "_h", None) is not None
            and getattr(tangent_fn, "steady_tangent_of", None) is system):
        native = (system._h, system.scratch())        # the linear tangent ignores the base
    return build_block_jacobi(tangent_fn, x, system.n_elements,
                              system.n_nodes * system.ncu, colors, native=native,
                              mode=jv_mode, residual_fn=residual_fn, invert=invert, share=share,
                              scratch=scratch)


class CompositeManager:
    """Config 'composite' (driver.py:145-175): block-Jacobi plus reduced-basis
    deflation built from the most recent Newton updates, inactive until
    snapshots exist; `note_update` is the Newton callback, `build(x)` is
    called by newton_solve at every Newton step (solver.py:241)."""

    def __init__(self, system, block_jacobi, tangent_fn, rank=10, refresh=1):
        self.system, self.block_jacobi, self.tangent_fn = system, block_jacobi, tangent_fn
        self.rank, self.refresh = rank, max(1, refresh)
        self.snapshots, self._builds, self._rb = [], 0, None

    def note_update(self, x, d):
        self.snapshots.append(d.clone())
        self.snapshots = self.snapshots[-self.rank:]

    def build(self, x):
        from .solver import CompositePreconditioner, build_reduced_basis
        self._builds += 1
        if self.snapshots and (self._builds % self.refresh == 0 or self._rb is None):
            try:
                self._rb = build_reduced_basis(self.snapshots,
                                               lambda v: self.tangent_fn(x, v), rank=self.rank)
            except Exception:
                self._rb = None
        return CompositePreconditioner(self.block_jacobi, self._rb)


def make_preconditioner(system, kind, residual_fn, tangent_fn, state_vec, steady=True,
                        jv_mode="tangent", rb_rank=10, rb_refresh=1, scratch=None):
    """driver.py:178-198 (identity, mass, block_jacobi, composite).  ``scratch``:
    device memory the block-Jacobi build may use for its probed blocks."""
    if kind == "auto":
        kind = "block_jacobi" if steady else "mass"
    if kind == "identity":
        return None, None
    if kind == "mass":
        return MassPreconditioner(system), None
    if kind == "block_jacobi":
        return build_pde_block_jacobi(system, residual_fn, tangent_fn, state_vec, jv_mode,
                                      scratch=scratch), None
    if kind == "composite":
        bj = build_pde_block_jacobi(system, residual_fn, tangent_fn, state_vec, jv_mode,
                                    scratch=scratch)
        mgr = CompositeManager(system, bj, tangent_fn, rank=rb_rank, refresh=rb_refresh)
        return mgr, mgr.note_update
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
        return system.tangent_dev(v.reshape(shape), base=uflat.reshape(shape),
                                  t=t).reshape(-1)

    import torch
    if getattr(system, "multi_block", False):
        def dev(a):
            return None if a is None else torch.as_tensor(
                a if isinstance(a, torch.Tensor) else np.ascontiguousarray(a, dtype=np.float64),
                device=system.device)
        x0 = system.pack(dev(state.u), dev(state.q), dev(state.w))
        x, stats = newton_solve(lambda Y: system.residual_packed_dev(Y, t), x0, opts,
                                precond=precond,
                                tangent_fn=lambda Y, V: system.tangent_packed_dev(V, Y, t),
                                callback=callback)
        u, q, w = system.unpack(x)
        return SolverState(u=u, q=q, w=w, t=t), stats
    u0 = state.u if isinstance(state.u, torch.Tensor) else torch.as_tensor(
        np.ascontiguousarray(state.u, dtype=np.float64), device=system.device)
    x, stats = newton_solve(residual, u0.reshape(-1).cuda(), opts, precond=precond,
                            tangent_fn=tangent, callback=callback)
    return SolverState(u=x.reshape(shape), q=None, w=None, t=t), stats


def run_steady(system, precond="block_jacobi", abs_tol=1e-11, rel_tol=3e-8, forcing=1e-8,
               restart=250, gmres_max_iter=6000, max_iter=20, orth="mgs", rb_rank=10,
               jv_mode="tangent"):
    """Steady branch of run_simulation (driver.py:253-268) with the
    acceptance solver flags as defaults; returns (state, stats, timings)."""
    import torch
    t0 = time.perf_counter()
    state = system.interpolate_initial_dev()
    res_fn, tan_fn = _steady_fns(system)
    u0 = torch.as_tensor(state.u, device=system.device).reshape(-1)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    scratch = None
    if precond in ("block_jacobi", "composite") and u0.is_cuda:
        # the first GMRES cycle's Krylov basis, allocated now (inside the timed
        # build) and lent to the block-Jacobi build for its probed blocks:
        # one multi-GB allocation in a fresh process instead of two
        from .solver import _WS
        m = min(restart, gmres_max_iter)
        scratch = _WS.get(m, u0.numel(), u0.device, need_z=orth != "dcgs2").V
    M, cb = make_preconditioner(system, precond, res_fn, tan_fn, u0, jv_mode=jv_mode,
                                rb_rank=rb_rank, scratch=scratch)
    del scratch
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    opts = NewtonOptions(abs_tol=abs_tol, rel_tol=rel_tol, max_iter=max_iter, forcing=forcing,
                         gmres_restart=restart, gmres_max_iter=gmres_max_iter,
                         jv_mode=jv_mode, orth=orth)
    out, stats = solve_steady(system, state, opts, precond=M, callback=cb)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    if not stats.converged:
        raise DriverError(f"steady Newton solve did not converge "
                          f"(residual {stats.final_residual:.3e})")
    tm = {"init_s": t1 - t0, "precond_build_s": t2 - t1, "solve_s": t3 - t2}
    if isinstance(M, BlockJacobiPreconditioner):
        tm["bj_blocks"] = M.nblk
        tm["bj_inverses"] = int(M.inv_t.shape[0])     # < bj_blocks: class-shared inverses
    return out, stats, tm


# ---------------------------------------------------------------------------
# DIRK time integration (timeint.py:33-207) on device vectors
# ---------------------------------------------------------------------------


class ButcherTableau:
    def __init__(self, A, b, c, order):
        self.A, self.b, self.c = (np.asarray(x, dtype=float) for x in (A, b, c))
        self.order = order

    @property
    def stages(self):
        return self.b.shape[0]

    @property
    def is_stiffly_accurate(self):
        return bool(np.allclose(self.A[-1], self.b, atol=1e-14))


def _alexander_gamma():
    """Root of x^3 - 3x^2 + 3x/2 - 1/6 in (1/6, 1/2) (timeint.py:73-85)."""
    x = 0.43
    for _ in range(60):
        f = x ** 3 - 3 * x ** 2 + 1.5 * x - 1 / 6
        step = f / (3 * x ** 2 - 6 * x + 1.5)
        x -= step
        if abs(step) < 1e-16:
            break
    if not (1 / 6 < x < 1 / 2):
        raise TimeIntError("SDIRK3 gamma iteration left (1/6, 1/2)")
    return x


def dirk_tableau(stages, order):
    """(1,1) implicit Euler, (2,2) L-stable SDIRK, (3,3) Alexander, (3,4)
    Crouzeix (timeint.py:88-112)."""
    if (stages, order) == (1, 1):
        return ButcherTableau([[1.0]], [1.0], [1.0], 1)
    if (stages, order) == (2, 2):
        g = 1.0 - 1.0 / np.sqrt(2.0)
        return ButcherTableau([[g, 0.0], [1.0 - g, g]], [1.0 - g, g], [g, 1.0], 2)
    if (stages, order) == (3, 3):
        g = _alexander_gamma()
        b1 = -1.5 * g ** 2 + 4.0 * g - 0.25
        b2 = 1.5 * g ** 2 - 5.0 * g + 1.25
        return ButcherTableau([[g, 0.0, 0.0], [(1.0 - g) / 2.0, g, 0.0], [b1, b2, g]],
                              [b1, b2, g], [g, (1.0 + g) / 2.0, 1.0], 3)
    if (stages, order) == (3, 4):
        g = 0.5 + np.cos(np.pi / 18.0) / np.sqrt(3.0)
        d = 1.0 / (6.0 * (2.0 * g - 1.0) ** 2)
        return ButcherTableau([[g, 0.0, 0.0], [0.5 - g, g, 0.0], [2.0 * g, 1.0 - 4.0 * g, g]],
                              [d, 1.0 - 2.0 * d, d], [g, 0.5, 1.0 - g], 4)
    raise TimeIntError(f"unsupported DIRK pair (stages={stages}, order={order}); "
                       "supported: (1,1),(2,2),(3,3),(3,4)")


class StepStats:
    def __init__(self):
        self.stage_stats = []

    @property
    def newton_iters(self):
        return sum(s.newton_iters for s in self.stage_stats)

    @property
    def gmres_iters(self):
        return sum(s.total_gmres_iters for s in self.stage_stats)

    @property
    def final_residual(self):
        return max((s.final_residual for s in self.stage_stats), default=0.0)


class StageSolveError(TimeIntError):
    def __init__(self, stage, stats):
        super().__init__(f"nonlinear solve failed at stage {stage} "
                         f"(residual {stats.final_residual:.3e})")
        self.stage, self.stats = stage, stats


def _stage_functions(system, Yk, a_dt, t_stage):
    """N(U) = M(U) (U - U_k)/(a dt) + R(U, t_i) and its tangent
    M(U) dU/(a dt) + (dM/dU dU)(U - U_k)/(a dt) + dR (timeint.py:132-165)."""
    shape = (system.n_elements, system.n_nodes, system.ncu)
    inv = 1.0 / a_dt
    if getattr(system, "multi_block", False):
        def stage_residual_p(Y):
            return system.mass_packed_dev(Y - Yk, Y, t_stage, inv) + \
                system.residual_packed_dev(Y, t_stage)

        def stage_tangent_p(Y, V):
            M = system.mass_packed_dev(V, Y, t_stage, inv)
            extra = system.mass_extra_packed_dev(Y - Yk, V, Y, t_stage, inv)
            if extra is not None:
                M = M + extra
            return M + system.tangent_packed_dev(V, Y, t_stage)

        return stage_residual_p, stage_tangent_p

    def stage_residual(Y):
        Ys = Y.reshape(shape)
        M = system.mass_apply_dev((Y - Yk).reshape(shape), scale=inv, base=Ys, t=t_stage)
        return (M + system.residual_dev(Ys, t_stage)).reshape(-1)

    def stage_tangent(Y, V):
        Ys, Vs = Y.reshape(shape), V.reshape(shape)
        M = system.mass_apply_dev(Vs, scale=inv, base=Ys, t=t_stage)
        extra = system.mass_tangent_extra_dev((Y - Yk).reshape(shape), Vs, Ys, t_stage,
                                              scale=inv)
        if extra is not None:
            M = M + extra
        return (M + system.tangent_dev(Vs, base=Ys, t=t_stage)).reshape(-1)

    return stage_residual, stage_tangent


def advance_step(system, state, dt, tableau, newton_options=None, precond=None, callback=None):
    """One DIRK step (timeint.py:168-207); state.u numpy or CUDA tensor."""
    import torch
    from .system import SolverState
    if dt <= 0:
        raise TimeIntError("dt must be positive")
    opts = newton_options or NewtonOptions()

    def dev(a):
        return None if a is None else (a if isinstance(a, torch.Tensor) else torch.as_tensor(
            np.ascontiguousarray(a, dtype=np.float64))).to(system.device)

    if getattr(system, "multi_block", False):
        Y0 = system.pack(dev(state.u), dev(state.q), dev(state.w)).clone()
    else:
        Y0 = dev(state.u).reshape(-1).clone()
    K, stats, Ylast = [], StepStats(), None
    for i in range(tableau.stages):
        Yk = Y0.clone()
        for j in range(i):
            Yk += dt * tableau.A[i, j] * K[j]
        a_dt = tableau.A[i, i] * dt
        t_stage = state.t + tableau.c[i] * dt
        res_fn, tan_fn = _stage_functions(system, Yk, a_dt, t_stage)
        guess = Yk + a_dt * K[-1] if K else Yk.clone()
        Yi, st = newton_solve(res_fn, guess, opts, precond=precond, tangent_fn=tan_fn,
                              callback=callback)
        stats.stage_stats.append(st)
        if not st.converged:
            raise StageSolveError(i, st)
        K.append((Yi - Yk) / a_dt)
        Ylast = Yi
    if tableau.is_stiffly_accurate:
        Ynew = Ylast
    else:
        Ynew = Y0.clone()
        for bi, Ki in zip(tableau.b, K):
            Ynew += dt * bi * Ki
    if not bool(torch.isfinite(Ynew).all()):
        raise TimeIntError("non-finite state after time step")
    if getattr(system, "multi_block", False):
        u, q, w = system.unpack(Ynew)
        return SolverState(u=u, q=q, w=w, t=state.t + dt), stats
    shape = (system.n_elements, system.n_nodes, system.ncu)
    return SolverState(u=Ynew.reshape(shape), q=None, w=None, t=state.t + dt), stats
