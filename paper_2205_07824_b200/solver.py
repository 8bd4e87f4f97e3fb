"""Device-resident Jacobian-free Newton-GMRES and the element block-Jacobi
preconditioner (mirrors ``ldgkit/solver.py``).

Vectors are flat float64 CUDA tensors in the reference's packed layout;
every O(n) operation is one of libldgb200's kernels (deterministic
warp-shuffle reductions, fused MGS sweeps, batched block inverses).  The
O(restart^2) Hessenberg / Givens / triangular-solve work stays on the host in
fp64 exactly as the reference does it, fed by one small device->host copy
per iteration.

Signatures and semantics follow the reference:
``gmres`` (solver.py:79-174), ``jacobian_vector`` (:193-212),
``newton_solve`` (:220-283), ``build_block_jacobi`` (:303-346),
``greedy_coloring`` / ``distance2_coloring`` (:355-378).
``orth="mgs"`` (default) reproduces the reference's modified Gram-Schmidt
with one conditional reorthogonalisation pass (the iteration-count parity
mode); ``orth="cgs2"`` is the fast block variant (two classical passes, two
multi-dot sweeps instead of 2(k+1) dependent ones); ``orth="cgs"`` takes the
second classical pass only under the reference's own reorthogonalisation
rule (||w|| < 0.707 ||w_before||), halving the Krylov traffic when the first
pass keeps orthogonality.
"""

from __future__ import annotations

from dataclasses import dataclass, field
import os

import numpy as np
import scipy.linalg

from . import _lib


class SolverError(RuntimeError):
    pass


@dataclass
class LinearOperator:
    apply: callable
    n: int
    matvecs: int = 0

    def __call__(self, v):
        self.matvecs += 1
        return self.apply(v)


@dataclass
class GmresResult:
    x: object
    converged: bool
    iterations: int
    residual_norms: list
    breakdown: bool = False


@dataclass
class SolveStats:
    newton_iters: int = 0
    residual_norms: list = field(default_factory=list)
    gmres_iters: list = field(default_factory=list)
    final_residual: float = 0.0
    converged: bool = False

    @property
    def total_gmres_iters(self):
        return int(sum(self.gmres_iters))


@dataclass
class NewtonOptions:
    abs_tol: float = 1e-8
    rel_tol: float = 1e-6
    max_iter: int = 20
    line_search: bool = True
    forcing: float | None = None
    gmres_restart: int = 30
    gmres_max_iter: int = 200
    jv_mode: str = "fd"
    orth: str = "mgs"


class IdentityPreconditioner:
    def apply(self, r):
        return r


# ---------------------------------------------------------------------------
# vector kernels
# ---------------------------------------------------------------------------


class VecOps:
    """Thin wrappers over the Krylov primitives of libldgb200 on the
    current stream.  Scalars live in a small device buffer; `host()` pulls
    them in one copy."""

    def __init__(self, device):
        import torch
        self.lib = _lib.load()
        self.device = device
        self.scratch = torch.empty(int(self.lib.ldg_reduce_scratch_doubles()),
                                   dtype=torch.float64, device=device)
        self.scratch.zero_()
        self.s = torch.zeros(8, dtype=torch.float64, device=device)

    def _st(self):
        return _lib.stream_ptr()

    def dot(self, x, y, out):
        _lib.check(self.lib.ldg_dot(x.numel(), _lib.ptr(x), _lib.ptr(y), _lib.ptr(self.scratch),
                                    _lib.ptr(out), self._st()), "ldg_dot")

    def nrm2(self, x, out):
        _lib.check(self.lib.ldg_nrm2(x.numel(), _lib.ptr(x), _lib.ptr(self.scratch),
                                     _lib.ptr(out), self._st()), "ldg_nrm2")

    def norm(self, x):
        self.nrm2(x, self.s[0:1])
        return float(self.s[0].item())

    def amax(self, x):
        """max |x_i| (host float); NaN propagates."""
        return float(x.abs().max().item()) if x.numel() else 0.0

    def axpy(self, a, x, y, a_dev=None, sign=1.0):
        _lib.check(self.lib.ldg_axpy(x.numel(), float(a), _lib.ptr(a_dev), float(sign),
                                     _lib.ptr(x), _lib.ptr(y), self._st()), "ldg_axpy")

    def div(self, x, den_dev, out):
        _lib.check(self.lib.ldg_div_scalar(x.numel(), _lib.ptr(x), _lib.ptr(den_dev),
                                           _lib.ptr(out), self._st()), "ldg_div_scalar")

    def div_guarded(self, x, den_dev, thr, out):
        _lib.check(self.lib.ldg_div_scalar_guarded(x.numel(), _lib.ptr(x), _lib.ptr(den_dev),
                                                   float(thr), _lib.ptr(out), self._st()),
                   "ldg_div_scalar_guarded")

    def mgs_step(self, vi, h_in, w, vnext, h_out):
        _lib.check(self.lib.ldg_mgs_step(w.numel(), _lib.ptr(vi), _lib.ptr(h_in), _lib.ptr(w),
                                         _lib.ptr(vnext), _lib.ptr(self.scratch),
                                         _lib.ptr(h_out), self._st()), "ldg_mgs_step")

    def cgs_dots(self, V, k, w, h):
        _lib.check(self.lib.ldg_cgs_dots(w.numel(), k, _lib.ptr(V), V.stride(0), _lib.ptr(w),
                                         _lib.ptr(self.scratch), _lib.ptr(h), self._st()),
                   "ldg_cgs_dots")

    def cgs_update(self, V, k, h, w, nrm_out):
        _lib.check(self.lib.ldg_cgs_update(w.numel(), k, _lib.ptr(V), V.stride(0), _lib.ptr(h),
                                           _lib.ptr(w), _lib.ptr(self.scratch),
                                           _lib.ptr(nrm_out), self._st()), "ldg_cgs_update")

    def dcgs_dots(self, V, k, x, y, hx, hy):
        _lib.check(self.lib.ldg_dcgs_dots(x.numel(), k, _lib.ptr(V), V.stride(0), _lib.ptr(x),
                                          _lib.ptr(y), _lib.ptr(self.scratch), _lib.ptr(hx),
                                          _lib.ptr(hy), self._st()), "ldg_dcgs_dots")

    def dcgs_update(self, V, m, s, t, v, w, out, inv_alpha, gamma, nrm_out):
        _lib.check(self.lib.ldg_dcgs_update(w.numel(), m, _lib.ptr(V), V.stride(0), _lib.ptr(s),
                                            _lib.ptr(t), _lib.ptr(v), _lib.ptr(w), _lib.ptr(out),
                                            float(inv_alpha), float(gamma),
                                            _lib.ptr(self.scratch), _lib.ptr(nrm_out),
                                            self._st()), "ldg_dcgs_update")

    def combine(self, Z, k, y, x):
        _lib.check(self.lib.ldg_combine(x.numel(), k, _lib.ptr(Z), Z.stride(0), _lib.ptr(y),
                                        _lib.ptr(x), self._st()), "ldg_combine")


_VECOPS = {}


def vecops(device):
    key = str(device)
    if key not in _VECOPS:
        _VECOPS[key] = VecOps(device)
    return _VECOPS[key]


def _as_device(v, device=None):
    """Flat float64 tensor; torch tensors keep their device (the product
    passes CUDA tensors), numpy arrays go to the GPU."""
    import torch
    if isinstance(v, torch.Tensor):
        return v.reshape(-1).to(torch.float64).contiguous(), True
    dev = device or torch.device("cuda")
    return torch.as_tensor(np.ascontiguousarray(v, dtype=np.float64).ravel(),
                           device=dev), False


# ---------------------------------------------------------------------------
# GMRES
# ---------------------------------------------------------------------------


class _Workspace:
    def __init__(self):
        self.key = None

    def get(self, m, n, device, need_z=True):
        import torch
        if self.key != (m, n, str(device)):
            self.V = self.Z = None
            torch.cuda.empty_cache()
            self.V = torch.empty((m + 1, n), dtype=torch.float64, device=device)
            self.w = torch.empty(n, dtype=torch.float64, device=device)
            self.H = torch.zeros((m + 1, m + 2), dtype=torch.float64, device=device)  # row k = column k of H
            self.c = torch.zeros(m + 2, dtype=torch.float64, device=device)
            self.nrm = torch.zeros(4, dtype=torch.float64, device=device)
            # DCGS2 dot / coefficient vectors (k+1 <= m+1 entries each)
            self.dv = torch.zeros((4, m + 2), dtype=torch.float64, device=device)
            self.key = (m, n, str(device))
        if need_z and self.Z is None:           # DCGS2 keeps no Z (x += M^-1 (V y))
            self.Z = torch.empty((m, n), dtype=torch.float64, device=device)
        return self


_WS = _Workspace()


def _nvtx(name, like):
    """NVTX range around a solver phase on CUDA data (timeline tools name the
    GMRES cycles and the block-Jacobi build); a no-op context otherwise."""
    import contextlib
    import torch
    if isinstance(like, torch.Tensor) and like.is_cuda:
        return torch.cuda.nvtx.range(name)
    return contextlib.nullcontext()


def _trace(tag):
    """LDG_GMRES_TRACE=1: synchronized wall-clock marks (diagnostics only)."""
    import os
    import time
    if not os.environ.get("LDG_GMRES_TRACE"):
        return lambda *_: None
    import torch
    state = {"t": time.perf_counter(), "n": 0}

    def mark(name):
        torch.cuda.synchronize()
        t = time.perf_counter()
        if state["n"] < 6 or state["n"] % 50 == 0:
            print(f"[gmres trace] {name} #{state['n']}: {1e3 * (t - state['t']):.2f} ms", flush=True)
        state["t"], state["n"] = t, state["n"] + 1
    return mark


def gmres(op, rhs, precond=None, rel_tol=1e-8, restart=30, max_iter=200, x0=None,
          orth="mgs", ops=None):
    """Right-preconditioned restarted GMRES (solver.py:79-174) on device
    vectors.  numpy rhs -> numpy x; CUDA tensor rhs -> CUDA tensor x.
    `ops` overrides the vector-kernel backend (e.g. parallel.DistVecOps)."""
    import torch
    b, on_dev = _as_device(rhs)
    n = b.numel()
    dev = b.device
    ops = ops or vecops(dev)
    if not (0.0 < rel_tol < 1.0):
        raise SolverError("gmres: rel_tol must be in (0, 1)")
    M = precond or IdentityPreconditioner()
    apply_op = op if callable(op) else op.apply
    x = torch.zeros(n, dtype=torch.float64, device=dev) if x0 is None else \
        _as_device(x0, dev)[0].clone()
    bnorm = ops.norm(b)
    if not np.isfinite(bnorm):
        raise SolverError("gmres: rhs contains non-finite entries")

    def out(xv):
        return xv if on_dev else xv.cpu().numpy()

    if bnorm == 0.0:
        return GmresResult(x=out(torch.zeros_like(b)), converged=True, iterations=0,
                           residual_norms=[0.0])
    tol = rel_tol * bnorm
    if orth == "dcgs2":
        return _gmres_dcgs2(apply_op, M, b, x, x0 is not None, bnorm, tol, restart, max_iter,
                            ops, out)
    res_norms, total, breakdown = [], 0, False
    while total < max_iter:
        if total > 0 or x0 is not None:
            r = b - apply_op(x)
        else:
            r = b.clone()
        beta = ops.norm(r)
        res_norms.append(beta)
        if beta <= tol:
            return GmresResult(out(x), True, total, res_norms, breakdown)
        m = min(restart, max_iter - total)
        _tr = _trace("ws")
        ws = _WS.get(m, n, dev)
        _tr("ws")
        V, Z, w, Hd, cd, nr = ws.V, ws.Z, ws.w, ws.H, ws.c, ws.nrm
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        torch.div(r, beta, out=V[0])
        k_done = 0
        for k in range(m):
            _tr("it")
            z = M.apply(V[k])
            Z[k].copy_(z)
            w.copy_(apply_op(Z[k]))
            ops.nrm2(w, nr[0:1])
            col = Hd[k]                     # contiguous: device kernels index it linearly
            if orth in ("cgs2", "cgs"):
                # classical Gram-Schmidt passes (one multi-dot + one fused
                # update/norm each); "cgs" takes the second pass under the
                # reference's rule ||w|| < 0.707 ||w_before|| (solver.py:139-144)
                ops.cgs_dots(V, k + 1, w, col)
                ops.cgs_update(V, k + 1, col, w, nr[1:2])
                reorth = orth == "cgs2"
                if not reorth:
                    hn = nr[:2].cpu().numpy()
                    if not np.isfinite(hn[0]):
                        raise SolverError("gmres: operator returned non-finite values")
                    reorth = hn[1] < 0.707 * hn[0]
                src = nr[1:2]
                if reorth:
                    ops.cgs_dots(V, k + 1, w, cd)
                    ops.cgs_update(V, k + 1, cd, w, nr[2:3])
                    col[: k + 1] += cd[: k + 1]
                    src = nr[2:3]
                hv = torch.cat([col[: k + 1], src, nr[0:1]]).cpu().numpy()
                nrm_w, nb0 = hv[k + 1], hv[k + 2]
                if not np.isfinite(nb0):
                    raise SolverError("gmres: operator returned non-finite values")
                H[: k + 1, k] = hv[: k + 1]
            else:
                # modified Gram-Schmidt, dot of V_{i+1} fused into the axpy of V_i
                ops.mgs_step(None, None, w, V[0], col[0:1])
                for i in range(k + 1):
                    ops.mgs_step(V[i], col[i:i + 1], w, V[i + 1] if i < k else None,
                                 col[i + 1:i + 2] if i < k else None)
                ops.nrm2(w, nr[1:2])
                hn = nr[:2].cpu().numpy()
                if not np.isfinite(hn[0]):
                    raise SolverError("gmres: operator returned non-finite values")
                src = nr[1:2]
                if hn[1] < 0.707 * hn[0]:
                    ops.mgs_step(None, None, w, V[0], cd[0:1])
                    for i in range(k + 1):
                        ops.mgs_step(V[i], cd[i:i + 1], w, V[i + 1] if i < k else None,
                                     cd[i + 1:i + 2] if i < k else None)
                    col[: k + 1] += cd[: k + 1]
                    ops.nrm2(w, nr[2:3])
                    src = nr[2:3]
                hv = torch.cat([col[: k + 1], src]).cpu().numpy()
                H[: k + 1, k] = hv[: k + 1]
                nrm_w = hv[k + 1]
            H[k + 1, k] = nrm_w
            total += 1
            k_done = k + 1
            if H[k + 1, k] <= 1e-14 * max(bnorm, 1.0):
                breakdown = True
            else:
                ops.div(w, src, V[k + 1])
            for i in range(k):
                t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
                H[i, k] = t
            den = np.hypot(H[k, k], H[k + 1, k])
            if den == 0.0:
                cs[k], sn[k] = 1.0, 0.0
            else:
                cs[k], sn[k] = H[k, k] / den, H[k + 1, k] / den
            H[k, k] = den
            H[k + 1, k] = 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            res_norms.append(float(abs(g[k + 1])))
            if abs(g[k + 1]) <= tol or breakdown:
                break
        y = scipy.linalg.solve_triangular(H[:k_done, :k_done], g[:k_done])
        ops.combine(Z, k_done, torch.as_tensor(y, device=dev), x)
        if abs(g[k_done]) <= tol:
            return GmresResult(out(x), True, total, res_norms, breakdown)
        if breakdown:
            r = b - apply_op(x)
            ok = ops.norm(r) <= tol
            return GmresResult(out(x), ok, total, res_norms, True)
    return GmresResult(out(x), False, total, res_norms, breakdown)


def _givens_column(R, Hr, c, cs, sn, g):
    """Rotate column c of the raw Hessenberg into R (solver.py:153-167)."""
    R[: c + 2, c] = Hr[: c + 2, c]
    for i in range(c):
        t = cs[i] * R[i, c] + sn[i] * R[i + 1, c]
        R[i + 1, c] = -sn[i] * R[i, c] + cs[i] * R[i + 1, c]
        R[i, c] = t
    den = np.hypot(R[c, c], R[c + 1, c])
    if den == 0.0:
        cs[c], sn[c] = 1.0, 0.0
    else:
        cs[c], sn[c] = R[c, c] / den, R[c + 1, c] / den
    R[c, c] = den
    R[c + 1, c] = 0.0
    g[c + 1] = -sn[c] * g[c]
    g[c] = cs[c] * g[c]
    return abs(g[c + 1])


def _gmres_dcgs2(apply_op, M, b, x, have_x0, bnorm, tol, restart, max_iter, ops, out):
    """GMRES with DCGS2 orthogonalisation: classical Gram-Schmidt with the
    reorthogonalisation pass of basis vector k delayed into iteration k+1,
    so each iteration makes ONE dot sweep over V (the dots of the
    once-orthogonalised v'_k and of the new Krylov vector w' = A M^-1 v'_k)
    and ONE update sweep (finalising v_k and projecting w'), against two of
    each for CGS2.  The Arnoldi relation A M^-1 V = V H turns the correction
    of v'_k into corrections of the Hessenberg coefficients:
      s = V^T v'_k, alpha = sqrt(v'.v' - s.s), H[:k, k-1] += nu s,
      H[k, k-1] = nu alpha, v_k = (v' - V s) / alpha,
      h_j = (t_j - (H s)_j) / alpha, h_k = (gamma - (H s)_k) / alpha,
      w1 = (w' - V t - gamma v_k) / alpha,  gamma = (v'.w' - s.t) / alpha,
    with t = V^T w'.  Column k-1 is final one iteration later, so the
    residual test (and the reported iteration count) lags by one matvec.
    Z is not stored: x += M^-1 (V y) (M linear).  Same restart, tolerance,
    breakdown and non-finite rules as the reference loop (solver.py:79-174)."""
    import torch
    n = b.numel()
    dev = b.device

    def apply_op_into(dst, v):
        dst.copy_(apply_op(M.apply(v)).reshape(-1))

    res_norms, total, breakdown = [], 0, False
    while total < max_iter:
        if total > 0 or have_x0:
            r = b - apply_op(x)
        else:
            r = b.clone()
        beta = ops.norm(r)
        res_norms.append(beta)
        if beta <= tol:
            return GmresResult(out(x), True, total, res_norms, breakdown)
        m = min(restart, max_iter - total)
        ws = _WS.get(m, n, dev, need_z=False)
        V, w, nr = ws.V, ws.w, ws.nrm
        dx, dy, sd, td = ws.dv[0], ws.dv[1], ws.dv[2], ws.dv[3]
        # s | t go to the device in one pinned copy per iteration (the stream
        # has synchronised on the next dot read before the buffer is reused)
        st_h = torch.empty(2 * (m + 2), dtype=torch.float64, pin_memory=dev.type == "cuda")
        st_d = torch.empty(2 * (m + 2), dtype=torch.float64, device=dev)
        thr = 1e-14 * max(bnorm, 1.0)
        Hr = np.zeros((m + 1, m))
        R = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        torch.div(r, beta, out=V[0])
        nr.zero_()
        ncol, lucky = 0, False
        for k in range(m + 1):
            # one host round trip per iteration: the dots of this sweep and
            # the norm nu of the previous update (its breakdown test deferred
            # to here; the normalisation ran on the device only when nu > thr)
            if k < m:
                apply_op_into(w, V[k])
                ops.dcgs_dots(V, k + 1, V[k], w, dx, dy)
            else:                                   # finalise the last column only
                ops.dcgs_dots(V, k + 1, V[k], V[k], dx, dy)
            hv = torch.cat([dx[: k + 1], dy[: k + 1], nr[0:1]]).cpu().numpy()
            if not np.isfinite(hv).all():
                raise SolverError("gmres: operator returned non-finite values")
            if k:
                nu = float(hv[2 * k + 2])
                lucky = nu <= thr
                if lucky and k < m:
                    # exact breakdown: V[k] is final unnormalised, the operator
                    # is not applied to it (solver.py:142); redo the sweep
                    ops.dcgs_dots(V, k + 1, V[k], V[k], dx, dy)
                    hv = torch.cat([dx[: k + 1], dy[: k + 1], nr[0:1]]).cpu().numpy()
            if k == 0:
                s = np.zeros(0)
                alpha, nu = 1.0, 1.0
            else:
                s, vv = hv[:k], hv[k]
                alpha = 0.0 if lucky else float(np.sqrt(max(vv - float(s @ s), 0.0)))
                Hr[:k, k - 1] += nu * s
                Hr[k, k - 1] = nu * alpha
                if Hr[k, k - 1] <= thr:
                    breakdown = True
                ncol = k
                total += 1
                res = _givens_column(R, Hr, k - 1, cs, sn, g)
                res_norms.append(float(res))
                if res <= tol or breakdown or k == m:
                    break
            t, vw = hv[k + 1: 2 * k + 1], hv[2 * k + 1]
            Hs = Hr[: k + 1, :k] @ s
            gamma = (vw - float(s @ t)) / alpha
            Hr[:k, k] = (t - Hs[:k]) / alpha
            Hr[k, k] = (gamma - Hs[k]) / alpha
            if k:
                st_h[:k] = torch.from_numpy(np.ascontiguousarray(s))
                st_h[k:2 * k] = torch.from_numpy(np.ascontiguousarray(t))
                st_d[: 2 * k].copy_(st_h[: 2 * k], non_blocking=True)
            ops.dcgs_update(V, k, st_d[:k], st_d[k: 2 * k] if k else st_d[:0], V[k], w, V[k + 1],
                            1.0 / alpha, gamma, nr[0:1])
            ops.div_guarded(V[k + 1], nr[0:1], thr, V[k + 1])
        if ncol:
            y = scipy.linalg.solve_triangular(R[:ncol, :ncol], g[:ncol])
            u = w
            u.zero_()
            ops.combine(V, ncol, torch.as_tensor(y, device=dev), u)
            x = x + M.apply(u).reshape(-1)
        if abs(g[ncol]) <= tol:
            return GmresResult(out(x), True, total, res_norms, breakdown)
        if breakdown:
            r = b - apply_op(x)
            ok = ops.norm(r) <= tol
            return GmresResult(out(x), ok, total, res_norms, True)
    return GmresResult(out(x), False, total, res_norms, breakdown)


# ---------------------------------------------------------------------------
# Jacobian-vector products
# ---------------------------------------------------------------------------


def fd_epsilon(base, v, ops=None):
    """eps = sqrt(eps_mach) (1 + ||base||_inf) / ||v||_2 (solver.py:182-190).
    With a distributed ``ops`` (parallel.DistVecOps) both norms are global
    (allreduced sum of squares and max), so every rank perturbs by the same
    eps."""
    import torch
    if ops is not None and isinstance(v, torch.Tensor):
        vnorm = ops.norm(v)
        bmax = ops.amax(base)
    else:
        vnorm = float(torch.linalg.vector_norm(v)) if isinstance(v, torch.Tensor) else \
            float(np.linalg.norm(v))
        bmax = float(base.abs().max()) if isinstance(base, torch.Tensor) else \
            float(np.abs(base).max())
    if vnorm == 0.0:
        raise SolverError("jacobian_vector: zero direction")
    eps = np.sqrt(np.finfo(float).eps) * (1.0 + bmax) / vnorm
    if eps == 0.0 or not np.isfinite(eps):
        raise SolverError("jacobian_vector: step underflow")
    return float(eps)


def jacobian_vector(residual_fn, base, v, mode="fd", base_residual=None, tangent_fn=None,
                    ops=None):
    """solver.py:193-212.  ``ops`` (optional) makes the FD step size and the
    non-finite check global across ranks."""
    if mode == "tangent":
        if tangent_fn is None:
            raise SolverError("tangent mode requires tangent_fn")
        return tangent_fn(base, v)
    if mode != "fd":
        raise SolverError(f"unknown jacobian mode {mode!r}")
    eps = fd_epsilon(base, v, ops)
    r0 = residual_fn(base) if base_residual is None else base_residual
    r1 = residual_fn(base + eps * v)
    out = (r1 - r0) / eps
    import torch
    if isinstance(out, torch.Tensor):
        bad = torch.logical_not(torch.isfinite(out).all()).to(torch.float64).reshape(1)
        fin = (ops.amax(bad) if ops is not None else float(bad.item())) == 0.0
    else:
        fin = bool(np.isfinite(out).all())
    if not fin:
        raise SolverError("jacobian_vector: non-finite result")
    return out


# ---------------------------------------------------------------------------
# Newton
# ---------------------------------------------------------------------------


def newton_solve(residual_fn, x0, options=None, precond=None, tangent_fn=None,
                 callback=None, ops=None):
    """Inexact Newton with right-preconditioned GMRES (solver.py:220-283);
    x0 may be numpy (returns numpy) or a CUDA tensor."""
    import torch
    opts = options or NewtonOptions()
    x, on_dev = _as_device(x0)
    x = x.clone()
    ops = ops or vecops(x.device)
    stats = SolveStats()
    R = residual_fn(x)
    rnorm = ops.norm(R)
    r0norm = rnorm
    stats.residual_norms.append(rnorm)
    for _ in range(opts.max_iter):
        if rnorm <= opts.abs_tol or rnorm <= opts.rel_tol * r0norm:
            stats.converged = True
            break
        M = precond.build(x) if hasattr(precond, "build") else precond
        xb, Rb = x, R
        op = LinearOperator(apply=lambda v: jacobian_vector(
            residual_fn, xb, v, opts.jv_mode, base_residual=Rb, tangent_fn=tangent_fn,
            ops=ops), n=x.numel())
        eta = opts.forcing if opts.forcing is not None else min(0.1, np.sqrt(rnorm))
        eta = min(max(eta, 1e-14), 0.9)
        with _nvtx(f"gmres (newton step {stats.newton_iters})", x):
            lin = gmres(op, -R, precond=M, rel_tol=eta, restart=opts.gmres_restart,
                        max_iter=opts.gmres_max_iter, orth=opts.orth, ops=ops)
        stats.gmres_iters.append(lin.iterations)
        d = lin.x
        step, accepted = 1.0, False
        for _ in range(9):
            x_trial = x + step * d
            R_trial = residual_fn(x_trial)
            rt = ops.norm(R_trial)
            if np.isfinite(rt) and (not opts.line_search or rt <= (1.0 - 1e-4 * step) * rnorm
                                    or rt <= opts.abs_tol):
                accepted = True
                break
            if not opts.line_search:
                break
            step *= 0.5
        stats.newton_iters += 1
        if not accepted:
            if np.isfinite(rt) and rt < rnorm:
                x, R, rnorm = x_trial, R_trial, rt
                stats.residual_norms.append(rnorm)
            break
        x, R, rnorm = x_trial, R_trial, rt
        stats.residual_norms.append(rnorm)
        if callback is not None:
            callback(x, d)
    if rnorm <= opts.abs_tol or rnorm <= opts.rel_tol * r0norm:
        stats.converged = True
    stats.final_residual = rnorm
    del torch
    return (x if on_dev else x.cpu().numpy()), stats


# ---------------------------------------------------------------------------
# block-Jacobi
# ---------------------------------------------------------------------------


class BlockJacobiPreconditioner:
    """z_b = A_b^-1 r_b per element block (solver.py:291-300); the inverses
    are stored transposed on the device.  ``perm`` (packed kind-W / ODE
    systems): perm[e*bs + j] = packed index of row j of element e's block
    (driver.py:128-142), gathered / scattered by native kernels."""

    def __init__(self, inv_t, bs, shifted=None, perm=None, classes=None):
        import torch
        self.inv_t, self.bs = inv_t, bs
        self.shifted = shifted
        self.perm = perm
        self.lib = _lib.load()
        self.classes = classes
        if classes is None:
            self.nblk = inv_t.shape[0]
            return
        self.nblk = int(classes.numel())
        self.tile_cls, self.tile_el = class_tiles(classes, inv_t.shape[0],
                                                  int(self.lib.ldg_bj_tile_elems()))
        self.ntiles = int(self.tile_cls.numel())

    def _apply_blocks(self, r, z, st):
        if self.classes is None:
            _lib.check(self.lib.ldg_bj_apply(self.nblk, self.bs, _lib.ptr(self.inv_t),
                                             _lib.ptr(r), _lib.ptr(z), st), "ldg_bj_apply")
        else:
            _lib.check(self.lib.ldg_bj_apply_tiles(self.ntiles, self.bs, _lib.ptr(self.inv_t),
                                                   _lib.ptr(self.tile_cls), _lib.ptr(self.tile_el),
                                                   _lib.ptr(r), _lib.ptr(z), st),
                       "ldg_bj_apply_tiles")

    def apply(self, r):
        import torch
        rd, dev = _as_device(r)
        z = torch.empty_like(rd)
        st = _lib.stream_ptr()
        if self.perm is None:
            self._apply_blocks(rd, z, st)
        else:
            re, ze = torch.empty_like(rd), torch.empty_like(rd)
            n = rd.numel()
            _lib.check(self.lib.ldg_permute_gather(n, _lib.ptr(self.perm), _lib.ptr(rd),
                                                   _lib.ptr(re), st), "ldg_permute_gather")
            self._apply_blocks(re, ze, st)
            _lib.check(self.lib.ldg_permute_scatter(n, _lib.ptr(self.perm), _lib.ptr(ze),
                                                    _lib.ptr(z), st), "ldg_permute_scatter")
        return z if dev else z.cpu().numpy()


def greedy_coloring(adjacency):
    """Deterministic greedy colouring (solver.py:355-365)."""
    n = len(adjacency)
    colors = -np.ones(n, dtype=int)
    for v in range(n):
        used = {colors[u] for u in adjacency[v] if colors[u] >= 0}
        c = 0
        while c in used:
            c += 1
        colors[v] = c
    return colors


def distance2_coloring(neighbors):
    """Colouring of the squared adjacency graph (solver.py:368-378)."""
    adj2 = []
    for v in range(len(neighbors)):
        s = set()
        for u in neighbors[v]:
            s.add(u)
            s |= neighbors[u]
        s.discard(v)
        adj2.append(s)
    return greedy_coloring(adj2)


def distance2_coloring_topology(topology, n_elements):
    """distance2_coloring(element_neighbor_sets(topology)) in the native
    library (same greedy order and result; linear time instead of Python
    set algebra over ~10^5 elements)."""
    import ctypes as C
    lib = _lib.load(require_gpu=False)
    el = np.ascontiguousarray(topology.elem_l, dtype=np.int32)
    er = np.ascontiguousarray(topology.elem_r, dtype=np.int32)
    out = np.empty(n_elements, dtype=np.int32)
    _lib.check(lib.ldg_color_distance2(n_elements, el.size, el.ctypes.data_as(C.c_void_p),
                                       er.ctypes.data_as(C.c_void_p),
                                       out.ctypes.data_as(C.c_void_p)), "ldg_color_distance2")
    return out.astype(np.int64)


def element_neighbor_sets(topology, n_elements):
    """driver.py:109-116."""
    nb = [set() for _ in range(n_elements)]
    for a, b in zip(np.asarray(topology.elem_l).tolist(), np.asarray(topology.elem_r).tolist()):
        nb[a].add(b)
        nb[b].add(a)
    return nb


def build_block_jacobi(tangent_fn, state, n_blocks, bs, colors, native=None, perm=None,
                       mode="tangent", residual_fn=None, base_residual=None, all_colors=None,
                       invert="auto", share=True, scratch=None):
    """Exact diagonal blocks by coloured unit probes (solver.py:303-346):
    colours x bs device Jacobian-vector products (``mode`` "tangent" through
    ``tangent_fn``, "fd" through ``residual_fn`` like jacobian_vector), then
    batched Gauss-Jordan inverses with the reference's 1e-12 shift rule.
    ``native`` = (handle, scratch) runs a colour's probes in one C call
    (only for the handle's own linear tangent); ``perm`` maps element-major
    block rows to packed indices (kind W / ODE systems).  ``share``: blocks
    that are bit-identical (structured meshes) are inverted once and applied
    per class (_block_classes; same z bit for bit).  ``all_colors``
    (partitioned systems): probe colours 0..all_colors-1 even where this
    rank owns no element of a colour, so the ranks' halo exchanges pair."""
    import torch
    lib = _lib.load()
    x, _ = _as_device(state)
    dev = x.device
    colors = np.asarray(colors, dtype=np.int64)
    if scratch is not None and scratch.is_cuda and scratch.dtype == torch.float64 and \
            scratch.numel() >= n_blocks * bs * bs and scratch.device == dev:
        # borrowed device memory (run_steady lends the Krylov basis, unused
        # until GMRES starts): no multi-GB allocation of its own
        mats = scratch.reshape(-1)[:n_blocks * bs * bs].view(n_blocks, bs, bs)
        mats.zero_()
    else:
        mats = torch.zeros((n_blocks, bs, bs), dtype=torch.float64, device=dev)
    v = torch.empty(n_blocks * bs, dtype=torch.float64, device=dev)
    st = _lib.stream_ptr()
    if mode == "fd":
        if residual_fn is None:
            raise SolverError("fd block-Jacobi probing needs residual_fn")
        R0 = residual_fn(x) if base_residual is None else base_residual
    elif mode != "tangent":
        raise SolverError(f"unknown jacobian mode {mode!r}")
    if perm is not None:
        vp = torch.empty_like(v)
        ce = torch.empty_like(v)

    def probe(vec):
        if mode == "tangent":
            return tangent_fn(x, vec)
        return jacobian_vector(residual_fn, x, vec, "fd", base_residual=R0)

    for c in (np.unique(colors) if all_colors is None else range(all_colors)):
        members = torch.as_tensor(np.nonzero(colors == c)[0].astype(np.int32), device=dev)
        if native is not None and perm is None and mode == "tangent":
            # linear fused / dense operator: the colour's bs probes in one C call
            h, scratch = native
            col = torch.empty_like(v)
            _lib.check(lib.ldg_bj_probe_colour(h, n_blocks, bs, _lib.ptr(members), members.numel(),
                                               _lib.ptr(v), _lib.ptr(col), _lib.ptr(scratch),
                                               _lib.ptr(mats), st), "ldg_bj_probe_colour")
            continue
        for k in range(bs):
            _lib.check(lib.ldg_bj_probe_vector(n_blocks, bs, _lib.ptr(members), members.numel(),
                                               k, _lib.ptr(v), st), "probe")
            if perm is None:
                col = probe(v)
            else:
                _lib.check(lib.ldg_permute_scatter(v.numel(), _lib.ptr(perm), _lib.ptr(v),
                                                   _lib.ptr(vp), st), "ldg_permute_scatter")
                colp = probe(vp).reshape(-1).contiguous()
                _lib.check(lib.ldg_permute_gather(v.numel(), _lib.ptr(perm), _lib.ptr(colp),
                                                  _lib.ptr(ce), st), "ldg_permute_gather")
                col = ce
            _lib.check(lib.ldg_bj_extract(bs, _lib.ptr(members), members.numel(), k,
                                          _lib.ptr(col), _lib.ptr(mats), st), "extract")
    classes = _block_classes(mats) if share else None
    if classes is not None:
        cls, reps = classes
        mats = mats[reps].contiguous()
    nb_inv = mats.shape[0]
    inv_t = torch.empty_like(mats)
    shifted = torch.zeros(nb_inv, dtype=torch.int32, device=dev)
    # blocks <= 160 in shared memory, larger ones (NS hex p=3: 320) on an
    # L2-resident global working copy; invert="global" forces the latter
    fn = lib.ldg_bj_invert_global if invert == "global" else lib.ldg_bj_invert
    _lib.check(fn(nb_inv, bs, _lib.ptr(mats), _lib.ptr(inv_t), _lib.ptr(shifted), st),
               "ldg_bj_invert")
    del mats
    if classes is not None:
        return BlockJacobiPreconditioner(inv_t, bs, shifted[cls], perm=perm, classes=cls)
    return BlockJacobiPreconditioner(inv_t, bs, shifted, perm=perm)


def class_tiles(classes, nclass, E):
    """Element tiles of one class each for ldg_bj_apply_tiles: (class per
    tile, E element ids per tile, -1 padded), elements in increasing order
    within a class.  Host index arithmetic (numpy), uploaded once."""
    import torch
    dev = classes.device if isinstance(classes, torch.Tensor) else torch.device("cpu")
    cls = classes.cpu().numpy() if isinstance(classes, torch.Tensor) else np.asarray(classes)
    n = cls.size
    order = np.argsort(cls, kind="stable")
    cs = cls[order]
    counts = np.bincount(cs, minlength=nclass)
    starts = np.cumsum(counts) - counts
    ntile_c = (counts + E - 1) // E
    tile_cls = np.repeat(np.arange(nclass), ntile_c)
    first = np.cumsum(ntile_c) - ntile_c                      # first tile of each class
    pos = np.arange(n) - starts[cs]                           # rank within the class
    slot = (first[cs] + pos // E) * E + pos % E
    tile_el = np.full(int(ntile_c.sum()) * E, -1, dtype=np.int32)
    tile_el[slot] = order
    return (torch.as_tensor(tile_cls.astype(np.int32), device=dev),
            torch.as_tensor(tile_el, device=dev))


BJ_SHARE_MAX_FRACTION = 0.125   # share inverses when classes <= 1/8 of the blocks


def _block_classes(mats):
    """Classes of bit-identical blocks (structured meshes: every interior
    element of one geometry class probes to the same block, bit for bit):
    exact keys of the blocks' bit patterns (device: ldg_bj_block_keys, two
    wrapping 64-bit sums; host: the bit rows themselves), grouped on the
    host, then on the device every block is compared with its class
    representative (ldg_bj_class_verify) -- any mismatch (a key collision)
    and no sharing.  Returns (class per block, representative block per
    class) as tensors on the blocks' device, or None when sharing would not
    pay.  No torch sort / unique kernels: their first use costs a few
    hundred ms of module loading in a fresh process."""
    import torch
    nblk = mats.shape[0]
    if nblk < 64:
        return None
    flat = mats.reshape(nblk, -1)
    if mats.is_cuda:
        lib = _lib.load()
        keys = torch.empty((nblk, 2), dtype=torch.int64, device=mats.device)
        _lib.check(lib.ldg_bj_block_keys(nblk, mats.shape[1], _lib.ptr(mats), _lib.ptr(keys),
                                         _lib.stream_ptr()), "ldg_bj_block_keys")
        kh = keys.cpu().numpy()
    else:
        kh = flat.numpy().view(np.int64)
    rows = np.ascontiguousarray(kh).view(np.dtype((np.void, kh.shape[1] * 8))).ravel()
    _, reps, cls = np.unique(rows, return_index=True, return_inverse=True)
    cls = cls.reshape(-1)
    if reps.size > BJ_SHARE_MAX_FRACTION * nblk:
        return None
    if mats.is_cuda:
        rep_of = torch.as_tensor(reps[cls].astype(np.int64), device=mats.device)
        bad = torch.zeros(1, dtype=torch.int32, device=mats.device)
        _lib.check(lib.ldg_bj_class_verify(nblk, mats.shape[1], _lib.ptr(mats), _lib.ptr(rep_of),
                                           _lib.ptr(bad), _lib.stream_ptr()), "ldg_bj_class_verify")
        if int(bad.item()):
            return None
    dev = mats.device
    return (torch.as_tensor(cls.astype(np.int64), device=dev),
            torch.as_tensor(reps.astype(np.int64), device=dev))


# ---------------------------------------------------------------------------
# Reduced-basis deflation and the composite preconditioner (solver.py:386-436)
# ---------------------------------------------------------------------------


class ReducedBasisPreconditioner:
    """apply(r) = W H^-1 W^T r + (I - W W^T) r with H = W^T J W
    (solver.py:386-399).  W is held as rows (rank x n) so W^T r is one
    multi-dot sweep and W (y - c) one fused combine; H's LU stays on the host
    (rank <= 10) like the reference's scipy lu_solve."""

    def __init__(self, W_rows, H_lu):
        import torch
        self.W = W_rows
        self._H_lu = H_lu
        self._c = torch.empty(W_rows.shape[0], dtype=torch.float64, device=W_rows.device)

    @property
    def rank(self):
        return self.W.shape[0]

    def apply(self, r):
        import torch
        ops = vecops(r.device)
        k = self.rank
        ops.cgs_dots(self.W, k, r, self._c)                  # c = W^T r
        c = self._c.cpu().numpy()
        y = scipy.linalg.lu_solve(self._H_lu, c) - c
        out = r.clone()
        ops.combine(self.W, k, torch.as_tensor(y, device=r.device), out)
        return out


def build_reduced_basis(snapshots, op, rank=None, drop_tol=1e-10, ops=None):
    """Orthonormalise the snapshots, H = W^T (J W) through the matrix-free
    operator, rank-deficient directions dropped (solver.py:402-423).  The
    reference's Householder QR is replaced by classical Gram-Schmidt with a
    second pass on the device vector kernels (ldg_cgs_dots / ldg_cgs_update /
    ldg_nrm2; allreduced through ``ops`` on partitioned systems): the same
    R diagonal |R_jj| (the norm of s_j's component orthogonal to the earlier
    snapshots) decides what is dropped, and W H^-1 W^T and W W^T do not depend
    on which orthonormal basis of the span is taken (column signs included)."""
    import torch
    if len(snapshots) == 0:
        raise SolverError("reduced basis needs at least one snapshot")
    snaps = [s.reshape(-1) for s in snapshots]
    if rank is not None:
        snaps = snaps[-rank:]
    dev = snaps[0].device
    ops = ops or vecops(dev)
    k, n = len(snaps), snaps[0].numel()
    Q = torch.empty((k, n), dtype=torch.float64, device=dev)
    h = torch.zeros(max(k, 1), dtype=torch.float64, device=dev)
    h2 = torch.zeros_like(h)
    nr = torch.zeros(2, dtype=torch.float64, device=dev)
    rdiag = np.zeros(k)
    for j in range(k):
        w = Q[j]
        w.copy_(snaps[j])
        if j:
            ops.cgs_dots(Q, j, w, h)
            ops.cgs_update(Q, j, h, w, None)
            ops.cgs_dots(Q, j, w, h2)                   # reorthogonalisation pass
            ops.cgs_update(Q, j, h2, w, None)
        ops.nrm2(w, nr[0:1])
        rdiag[j] = float(nr[0].item())
        if rdiag[j] > 0.0:
            ops.div(w, nr[0:1], w)
    keep = rdiag > drop_tol * max(1.0, float(rdiag.max()))
    if not keep.any():
        raise SolverError("all snapshot directions are degenerate")
    W = Q[torch.as_tensor(np.nonzero(keep)[0], device=dev)].contiguous()
    apply_op = op if callable(op) else op.apply
    r = W.shape[0]
    H = np.zeros((r, r))
    hc = torch.zeros(r, dtype=torch.float64, device=dev)
    for c in range(r):
        jw = apply_op(W[c]).reshape(-1).contiguous()
        ops.cgs_dots(W, r, jw, hc)                      # column c of W^T J W
        H[:, c] = hc.cpu().numpy()
    return ReducedBasisPreconditioner(W, scipy.linalg.lu_factor(H))


class CompositePreconditioner:
    """Block-Jacobi, then the reduced-basis deflation (solver.py:426-436)."""

    def __init__(self, block_jacobi, reduced_basis=None):
        self.block_jacobi = block_jacobi
        self.reduced_basis = reduced_basis

    def apply(self, r):
        z = self.block_jacobi.apply(r)
        if self.reduced_basis is not None:
            z = self.reduced_basis.apply(z)
        return z
