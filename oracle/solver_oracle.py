"""ORACLE -- test infrastructure only, never imported by the product path.

numpy restatement of the reference's matrix-free Newton-GMRES and block-Jacobi
preconditioner (``ldgkit/solver.py``), used to check iteration counts,
residual histories and converged solutions of the device solver.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg


def gmres(op, rhs, precond=None, rel_tol=1e-8, restart=30, max_iter=200, x0=None):
    """Right-preconditioned restarted GMRES, MGS + one conditional
    reorthogonalisation pass, Givens updates (solver.py:79-174).  Returns
    (x, converged, iterations, residual_norms, breakdown)."""
    rhs = np.asarray(rhs, dtype=float)
    n = rhs.shape[0]
    M = precond if precond is not None else (lambda r: r)
    x = np.zeros(n) if x0 is None else np.asarray(x0, dtype=float).copy()
    bnorm = np.linalg.norm(rhs)
    if bnorm == 0.0:
        return np.zeros(n), True, 0, [0.0], False
    tol = rel_tol * bnorm
    hist, total, brk = [], 0, False
    while total < max_iter:
        r = rhs - op(x) if (total > 0 or x0 is not None) else rhs.copy()
        beta = np.linalg.norm(r)
        hist.append(float(beta))
        if beta <= tol:
            return x, True, total, hist, brk
        m = min(restart, max_iter - total)
        V = np.zeros((m + 1, n))
        Z = np.zeros((m, n))
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        kd = 0
        for k in range(m):
            Z[k] = M(V[k])
            w = op(Z[k])
            n0 = np.linalg.norm(w)
            for i in range(k + 1):
                H[i, k] = np.dot(V[i], w)
                w = w - H[i, k] * V[i]
            if np.linalg.norm(w) < 0.707 * n0:
                for i in range(k + 1):
                    c = np.dot(V[i], w)
                    H[i, k] += c
                    w = w - c * V[i]
            H[k + 1, k] = np.linalg.norm(w)
            total += 1
            kd = k + 1
            if H[k + 1, k] <= 1e-14 * max(bnorm, 1.0):
                brk = True
            else:
                V[k + 1] = w / H[k + 1, k]
            for i in range(k):
                tt = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
                H[i, k] = tt
            den = np.hypot(H[k, k], H[k + 1, k])
            if den == 0.0:
                cs[k], sn[k] = 1.0, 0.0
            else:
                cs[k], sn[k] = H[k, k] / den, H[k + 1, k] / den
            H[k, k] = den
            H[k + 1, k] = 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            hist.append(float(abs(g[k + 1])))
            if abs(g[k + 1]) <= tol or brk:
                break
        y = scipy.linalg.solve_triangular(H[:kd, :kd], g[:kd])
        x = x + Z[:kd].T @ y
        if abs(g[kd]) <= tol:
            return x, True, total, hist, brk
        if brk:
            return x, bool(np.linalg.norm(rhs - op(x)) <= tol), total, hist, True
    return x, False, total, hist, brk


def newton_solve(residual_fn, tangent_fn, x0, abs_tol=1e-8, rel_tol=1e-6,
                 max_iter=20, forcing=None, restart=30, gmres_max_iter=200,
                 precond=None, line_search=True):
    """Inexact Newton with backtracking (solver.py:220-283).  Returns
    (x, dict(newton_iters, gmres_iters, residual_norms, converged))."""
    x = np.asarray(x0, dtype=float).copy()
    R = residual_fn(x)
    rn = float(np.linalg.norm(R))
    r0 = rn
    st = {"newton_iters": 0, "gmres_iters": [], "residual_norms": [rn],
          "converged": False}
    for _ in range(max_iter):
        if rn <= abs_tol or rn <= rel_tol * r0:
            st["converged"] = True
            break
        eta = forcing if forcing is not None else min(0.1, np.sqrt(rn))
        eta = min(max(eta, 1e-14), 0.9)
        d, _, its, _, _ = gmres(lambda v: tangent_fn(x, v), -R, precond, eta,
                                restart, gmres_max_iter)
        st["gmres_iters"].append(its)
        step, ok = 1.0, False
        for _ in range(9):
            xt = x + step * d
            Rt = residual_fn(xt)
            rt = float(np.linalg.norm(Rt))
            if np.isfinite(rt) and (not line_search or rt <= (1.0 - 1e-4 * step) * rn
                                    or rt <= abs_tol):
                ok = True
                break
            if not line_search:
                break
            step *= 0.5
        st["newton_iters"] += 1
        if not ok:
            if np.isfinite(rt) and rt < rn:
                x, R, rn = xt, Rt, rt
                st["residual_norms"].append(rn)
            break
        x, R, rn = xt, Rt, rt
        st["residual_norms"].append(rn)
    if rn <= abs_tol or rn <= rel_tol * r0:
        st["converged"] = True
    st["final_residual"] = rn
    return x, st


def greedy_coloring(adj):
    """solver.py:355-365."""
    col = -np.ones(len(adj), dtype=int)
    for v in range(len(adj)):
        used = {col[u] for u in adj[v] if col[u] >= 0}
        c = 0
        while c in used:
            c += 1
        col[v] = c
    return col


def distance2_coloring(nbrs):
    """solver.py:368-378."""
    adj2 = []
    for v in range(len(nbrs)):
        s = set()
        for u in nbrs[v]:
            s.add(u)
            s |= nbrs[u]
        s.discard(v)
        adj2.append(s)
    return greedy_coloring(adj2)


def element_neighbors(topo, ne):
    nb = [set() for _ in range(ne)]
    for a, b in zip(topo.elem_l.tolist(), topo.elem_r.tolist()):
        nb[a].add(b)
        nb[b].add(a)
    return nb


def block_jacobi_blocks(tangent_fn, x, ne, bs, colors):
    """Exact diagonal blocks by coloured unit probes (solver.py:303-334)."""
    mats = np.zeros((ne, bs, bs))
    for c in np.unique(colors):
        members = np.nonzero(colors == c)[0]
        for k in range(bs):
            v = np.zeros(ne * bs)
            v[members * bs + k] = 1.0
            col = tangent_fn(x, v).reshape(ne, bs)
            mats[members, :, k] = col[members]
    return mats


def block_jacobi_factor(mats):
    """Per-block LU with the reference's 1e-12 shift rule (solver.py:335-345)."""
    bs = mats.shape[1]
    lus = []
    for A in mats:
        try:
            lu = scipy.linalg.lu_factor(A)
            if not np.isfinite(lu[0]).all() or \
                    np.any(np.abs(np.diag(lu[0])) < 1e-14 * max(1, np.abs(A).max())):
                raise scipy.linalg.LinAlgError
        except (scipy.linalg.LinAlgError, ValueError):
            lu = scipy.linalg.lu_factor(A + 1e-12 * np.eye(bs))
        lus.append(lu)

    def apply(r):
        out = np.asarray(r, dtype=float).copy().reshape(len(lus), bs)
        for b, lu in enumerate(lus):
            out[b] = scipy.linalg.lu_solve(lu, out[b])
        return out.ravel()

    return apply
