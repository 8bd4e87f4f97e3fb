"""ORACLE -- test infrastructure only, never imported by the product path.

CPU restatement (numpy) of the reference LDG residual / Jacobian-vector
product path, following ``ldgkit/disc.py`` and ``ldgkit/expr.py`` function by
function (file:line cited on each).  It exists to check the CUDA path:
``tests/`` compare the B200 kernels against it on seeded inputs, and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs time it as the
reference CPU implementation (the reference package itself is pure Python
and cannot travel to the GPU box).

Parity pinning: ``tests/test_oracle_golden.py`` checks this module against
golden vectors produced by the *unmodified* reference package
(``tests/golden/gen_golden.py``, run in the build container where
``/root/reference`` is mounted): residuals, tangents, mixed gradients and
switch bits on hex/quad/tri/tet meshes.

Scope: kinds D and C with the default trace rules or user u^ / f^
overrides, dirichlet / neumann boundaries, constant or state-dependent mass.
Kind W and pointwise ODE blocks raise ``NotImplementedError`` (those device
paths are pinned directly against the reference's golden vectors).
"""

from __future__ import annotations

import numpy as np


class OracleNanError(ValueError):
    pass


# ---------------------------------------------------------------------------
# pointwise plans with forward tangents (expr.py:519-651)
# ---------------------------------------------------------------------------


def _fn(fn, a, b=None):
    if fn == "abs":
        return np.abs(a)
    if fn == "min":
        return np.minimum(a, b)
    if fn == "max":
        return np.maximum(a, b)
    if fn == "pow":
        return a ** b
    return getattr(np, fn)(a)


def _pow_dual(a, da, b, db):
    """expr.py:611-617: log term only where db != 0."""
    v = a ** b
    d = b * a ** (b - 1.0) * da
    if np.any(db != 0.0):
        d = d + np.where(db == 0.0, 0.0, v * np.log(a) * db)
    return v, d


def _unary_dual(fn, a, da):
    """expr.py:620-641."""
    if fn == "sin":
        return np.sin(a), np.cos(a) * da
    if fn == "cos":
        return np.cos(a), -np.sin(a) * da
    if fn == "tan":
        v = np.tan(a)
        return v, (1.0 + v * v) * da
    if fn == "exp":
        v = np.exp(a)
        return v, v * da
    if fn == "log":
        return np.log(a), da / a
    if fn == "sqrt":
        v = np.sqrt(a)
        return v, da / (2.0 * v)
    if fn == "abs":
        return np.abs(a), np.sign(a) * da
    if fn == "tanh":
        v = np.tanh(a)
        return v, (1.0 - v * v) * da
    raise AssertionError(fn)


def run_plan(plan, bind, seed=None):
    """Evaluate a plan (reference instruction tuples) over batch bindings;
    with `seed` also return forward tangents (expr.py:519-608)."""
    used = {ins[1] for ins in plan.instructions if ins[0] == "sym"}
    arrs, batch = {}, 1
    for s in used:
        if s not in bind:
            raise KeyError(f"missing binding {s}")
        a = np.asarray(bind[s], dtype=float).ravel()
        arrs[s] = a
        if a.shape[0] > 1:
            batch = max(batch, a.shape[0])
    zero = np.zeros(1)
    seed = {} if seed is None else {k: np.asarray(v, float).ravel()
                                     for k, v in seed.items()}
    vals, tans = [], []
    with np.errstate(all="ignore"):
        for ins in plan.instructions:
            tag = ins[0]
            if tag == "const":
                v, d = np.full(1, ins[1]), zero
            elif tag == "sym":
                v, d = arrs[ins[1]], seed.get(ins[1], zero)
            elif tag == "neg":
                v, d = -vals[ins[1]], -tans[ins[1]]
            elif tag == "call":
                fn, args = ins[1], ins[2]
                a, da = vals[args[0]], tans[args[0]]
                if fn in ("min", "max", "pow"):
                    b, db = vals[args[1]], tans[args[1]]
                    if fn == "min":
                        v, d = np.minimum(a, b), np.where(a <= b, da, db)
                    elif fn == "max":
                        v, d = np.maximum(a, b), np.where(a >= b, da, db)
                    else:
                        v, d = _pow_dual(a, da, b, db)
                else:
                    v, d = _unary_dual(fn, a, da)
            else:
                a, da = vals[ins[1]], tans[ins[1]]
                b, db = vals[ins[2]], tans[ins[2]]
                if tag == "add":
                    v, d = a + b, da + db
                elif tag == "sub":
                    v, d = a - b, da - db
                elif tag == "mul":
                    v, d = a * b, da * b + a * db
                elif tag == "div":
                    v = a / b
                    d = (da - v * db) / b
                else:
                    v, d = _pow_dual(a, da, b, db)
            vals.append(v)
            tans.append(d)
    out = np.empty((len(plan.outputs), batch))
    dout = np.empty((len(plan.outputs), batch))
    for k, r in enumerate(plan.outputs):
        out[k] = vals[r]
        dout[k] = tans[r]
    return out, (dout if seed is not None else None)


# ---------------------------------------------------------------------------
# geometry tables (disc.py:74-239)
# ---------------------------------------------------------------------------


def _face_normal_ref(kind, lf, face_map):
    _, T = face_map(kind, lf)
    if kind == "line":
        return np.array([-1.0]) if lf == 0 else np.array([1.0])
    if T.shape[1] == 2:
        n = np.array([T[0][1], -T[0][0]])
    else:
        n = np.cross(T[0], T[1])
    return n / np.linalg.norm(n)


class OracleDisc:
    """Per-quadrature-point metrics and dense trace tabulations, computed the
    reference way (disc.py:79-225): volume Jacobians from the geometry
    basis, face normals from tangent cross products, right tabulations by a
    per-face Newton inversion of the right element's map."""

    def __init__(self, mesh, topo, master, geom_master, face_map):
        self.mesh, self.topo, self.master = mesh, topo, master
        self.geom, self.face_map = geom_master, face_map
        ho = mesh.ho_nodes
        gphi = geom_master.eval_basis(master.quad_pts)
        gdphi = geom_master.eval_basis_grad(master.quad_pts)
        J = np.einsum("egd,qgr->eqdr", ho, gdphi)
        detj = np.linalg.det(J)
        if np.any(detj <= 0):
            raise ValueError("nonpositive Jacobian")
        self.detj = detj
        self.invjt = np.linalg.inv(J).transpose(0, 1, 3, 2)
        self.wdetj = master.quad_wts[None, :] * detj
        self.xq = np.einsum("qg,egd->eqd", gphi, ho)
        self.node_x = np.einsum("ng,egd->end", geom_master.eval_basis(master.nodes), ho)
        self.mass = np.einsum("eq,qa,qb->eab", self.wdetj, master.phi, master.phi)
        self.mass_inv = np.linalg.inv(self.mass)
        self._gfphi = [geom_master.eval_basis(f.xi) for f in master.faces]
        self._gfdphi = [geom_master.eval_basis_grad(f.xi) for f in master.faces]
        self.fi_x, self.fi_n, self.fi_wsj, self.fi_phi_l = \
            self._faces(topo.elem_l, topo.face_l)
        self.fi_phi_r = self._right_tabs()
        self.fb_x, self.fb_n, self.fb_wsj, self.fb_phi = \
            self._faces(topo.elem_b, topo.face_b)
        self.fi_nbar = self.fi_n.mean(axis=1)
        self.elem_vol = self.wdetj.sum(axis=1)
        fa = np.maximum(self.fi_wsj.sum(axis=1), 1e-300)
        fb = np.maximum(self.fb_wsj.sum(axis=1), 1e-300)
        self.fi_h = 0.5 * (self.elem_vol[topo.elem_l] + self.elem_vol[topo.elem_r]) / fa
        self.fb_h = self.elem_vol[topo.elem_b] / fb
        if mesh.nd == 1:
            self.fi_h = 0.5 * (self.elem_vol[topo.elem_l] + self.elem_vol[topo.elem_r])
            self.fb_h = self.elem_vol[topo.elem_b]

    def _faces(self, elems, lfs):
        """disc.py:139-180."""
        mesh, master = self.mesh, self.master
        nd, nf = mesh.nd, elems.shape[0]
        nqf = master.faces[0].weights.shape[0] if master.faces else 0
        x = np.zeros((nf, nqf, nd))
        n = np.zeros((nf, nqf, nd))
        wsj = np.zeros((nf, nqf))
        phi = np.zeros((nf, nqf, master.n_nodes))
        for lf in range(master.n_faces):
            sel = np.nonzero(lfs == lf)[0]
            if sel.size == 0:
                continue
            ho = mesh.ho_nodes[elems[sel]]
            x[sel] = np.einsum("qg,kgd->kqd", self._gfphi[lf], ho)
            phi[sel] = master.faces[lf].phi[None, :, :]
            w = master.faces[lf].weights
            if nd == 1:
                n[sel] = _face_normal_ref(mesh.elem_kind, lf, self.face_map)[None, None, :]
                wsj[sel] = w[None, :]
                continue
            _, T = self.face_map(mesh.elem_kind, lf)
            tang = np.einsum("qgd,sd,kgc->kqcs", self._gfdphi[lf], T, ho)
            if nd == 2:
                t = tang[:, :, :, 0]
                nv = np.stack([t[:, :, 1], -t[:, :, 0]], axis=-1)
            else:
                nv = np.cross(tang[:, :, :, 0], tang[:, :, :, 1])
            mag = np.linalg.norm(nv, axis=-1)
            n[sel] = nv / mag[:, :, None]
            wsj[sel] = w[None, :] * mag
        return x, n, wsj, phi

    def _right_tabs(self):
        """disc.py:182-225: Newton-invert the right element map at the left
        element's physical face points (periodic translation applied)."""
        mesh, master, topo = self.mesh, self.master, self.topo
        nfi, nqf = topo.elem_l.shape[0], self.fi_x.shape[1]
        out = np.zeros((nfi, nqf, master.n_nodes))
        if nfi == 0:
            return out
        target = self.fi_x + topo.translation[:, None, :]
        scale = max(mesh.diameter(), 1.0)
        for lf in range(master.n_faces):
            sel = np.nonzero(topo.face_r == lf)[0]
            if sel.size == 0:
                continue
            origin, T = self.face_map(mesh.elem_kind, lf)
            ho = mesh.ho_nodes[topo.elem_r[sel]]
            xt = target[sel]
            k = sel.size
            sig = np.tile(master.faces[lf].sigma.mean(axis=0), (k, nqf, 1))
            for _ in range(50):
                xi = origin[None, None, :] + sig @ T
                pts = xi.reshape(-1, mesh.nd)
                g = self.geom.eval_basis(pts).reshape(k, nqf, -1)
                gd = self.geom.eval_basis_grad(pts).reshape(k, nqf, -1, mesh.nd)
                res = xt - np.einsum("kqg,kgd->kqd", g, ho)
                if np.max(np.abs(res)) < 1e-13 * scale:
                    break
                tang = np.einsum("kqgd,sd,kgc->kqcs", gd, T, ho)
                A = np.einsum("kqcs,kqcr->kqsr", tang, tang)
                b = np.einsum("kqcs,kqc->kqs", tang, res)
                sig = sig + np.linalg.solve(A, b[..., None])[..., 0]
            else:
                raise ValueError("face inverse mapping did not converge")
            xi = origin[None, None, :] + sig @ T
            out[sel] = master.eval_basis(xi.reshape(-1, mesh.nd)).reshape(k, nqf, -1)
        return out

    def trace_l(self, a):
        return np.einsum("fqa,fa...->fq...", self.fi_phi_l, a[self.topo.elem_l])

    def trace_r(self, a):
        return np.einsum("fqa,fa...->fq...", self.fi_phi_r, a[self.topo.elem_r])

    def trace_b(self, a):
        return np.einsum("fqa,fa...->fq...", self.fb_phi, a[self.topo.elem_b])


def scatter_add(target, elems, vals):
    """Deterministic bincount accumulation (disc.py:242-249)."""
    ne = target.shape[0]
    m = int(np.prod(target.shape[1:]))
    idx = (elems[:, None] * m + np.arange(m)[None, :]).ravel()
    acc = np.bincount(idx, weights=vals.reshape(len(elems), m).ravel(),
                      minlength=ne * m)
    target += acc.reshape(target.shape)


# ---------------------------------------------------------------------------
# the semi-discrete operator (disc.py:257-948)
# ---------------------------------------------------------------------------


class OracleLdg:
    """Residual, tangent, mixed gradient and mass operator of the reference
    ``LdgSystem`` for kinds D and C."""

    def __init__(self, model, mesh, topo, master, geom_master, face_map):
        if model.kind == "W" or model.nw > 0:
            raise NotImplementedError("oracle covers kinds D and C without ODEs")

        self.model, self.mesh, self.topo, self.master = model, mesh, topo, master
        self.d = OracleDisc(mesh, topo, master, geom_master, face_map)
        self.kind, self.ncu, self.nd = model.kind, model.ncu, model.nd
        beta = np.ones(mesh.nd) / np.sqrt(mesh.nd)
        self.switch = (self.d.fi_nbar @ beta) > 0.0            # disc.py:285-287
        self.bc_groups = []
        tags = np.unique(topo.tag_b) if topo.elem_b.shape[0] else []
        for tag in tags:                                      # disc.py:289-304
            tag = int(tag)
            if tag not in model.bcs:
                raise ValueError(f"mesh boundary tag {tag} has no [bc] entry")
            bc = model.bcs[tag]
            if bc.type not in ("dirichlet", "neumann"):
                raise NotImplementedError(bc.type)
            self.bc_groups.append((tag, bc, np.nonzero(topo.tag_b == tag)[0]))
        self.mu = model.mu_bindings()
        self.mass_const = all(i[0] == "const" for i in model.mass_plan().instructions)

    @property
    def n_dofs(self):
        return self.mesh.connectivity.shape[0] * self.master.n_nodes * self.ncu

    # -- bindings ---------------------------------------------------------------
    def _bind(self, x, t, u=None, q=None, n=None):
        b = {"t": float(t)}
        b.update(self.mu)
        for k in range(self.nd):
            b[f"x{k + 1}"] = x[..., k].ravel()
        if u is not None:
            for i in range(self.ncu):
                b[f"u{i + 1}"] = u[..., i].ravel()
        if q is not None:
            for i in range(self.ncu):
                for j in range(self.nd):
                    b[f"q{i + 1}_{j + 1}"] = q[..., i, j].ravel()
        if n is not None:
            for k in range(self.nd):
                b[f"n{k + 1}"] = n[..., k].ravel()
        return b

    def _face_bind(self, x, t, ul, ur, ql, qr, n):
        """Face-override bindings over both traces (disc.py:516-547)."""
        b = {"t": float(t)}
        b.update(self.mu)
        for k in range(self.nd):
            b[f"x{k + 1}"] = x[..., k].ravel()
            b[f"n{k + 1}"] = n[..., k].ravel()
        for i in range(self.ncu):
            b[f"ul{i + 1}"] = ul[..., i].ravel()
            b[f"ur{i + 1}"] = ur[..., i].ravel()
        if ql is not None:
            for i in range(self.ncu):
                for j in range(self.nd):
                    b[f"ql{i + 1}_{j + 1}"] = ql[..., i, j].ravel()
                    b[f"qr{i + 1}_{j + 1}"] = qr[..., i, j].ravel()
        return b

    def _face_seed(self, dul, dur, dql, dqr):
        s = {}
        for i in range(self.ncu):
            s[f"ul{i + 1}"] = dul[..., i].ravel()
            s[f"ur{i + 1}"] = dur[..., i].ravel()
        if dql is not None:
            for i in range(self.ncu):
                for j in range(self.nd):
                    s[f"ql{i + 1}_{j + 1}"] = dql[..., i, j].ravel()
                    s[f"qr{i + 1}_{j + 1}"] = dqr[..., i, j].ravel()
        return s

    def _seed(self, du=None, dq=None):
        s = {}
        if du is not None:
            for i in range(self.ncu):
                s[f"u{i + 1}"] = du[..., i].ravel()
        if dq is not None:
            for i in range(self.ncu):
                for j in range(self.nd):
                    s[f"q{i + 1}_{j + 1}"] = dq[..., i, j].ravel()
        return s

    def _eval(self, plan, bind, shape, label, seed=None):
        """disc.py:393-416 (NaN check with element id)."""
        out, tan = run_plan(plan, bind, seed)
        if not np.isfinite(out).all():
            col = int(np.argwhere(~np.isfinite(out))[0][1])
            nq = shape[1] if len(shape) > 1 else 1
            raise OracleNanError(f"{label} kernel produced non-finite values "
                                 f"(first at element {col // nq})")
        no, B = out.shape[0], int(np.prod(shape))
        if out.shape[1] != B:
            out = np.broadcast_to(out, (no, B))
            if tan is not None:
                tan = np.broadcast_to(tan, (no, B))
        out = np.moveaxis(out.reshape((no,) + tuple(shape)), 0, -1)
        if tan is not None:
            tan = np.moveaxis(tan.reshape((no,) + tuple(shape)), 0, -1)
        return out, tan

    def interpolate_initial(self):
        ne, nb = self.d.node_x.shape[:2]
        v, _ = self._eval(self.model.init_plan(), self._bind(self.d.node_x, 0.0),
                          (ne, nb), "initial")
        return v[..., :self.ncu].copy()

    # -- mixed gradient (disc.py:436-574) -----------------------------------------
    def compute_mixed(self, u, t, homogeneous=False):
        rhs = self._lifted(u, t, homogeneous)
        return np.einsum("eab,ebij->eaij", self.d.mass_inv, rhs)

    def _lifted(self, u, t, homogeneous):
        d, m = self.d, self.master
        g = np.einsum("eai,eqjr,qar->eqij", u, d.invjt, m.dphi, optimize=True)
        rhs = -np.einsum("eq,eqij,qa->eaij", d.wdetj, g, m.phi, optimize=True)
        if self.topo.elem_l.shape[0]:
            ul, ur = d.trace_l(u), d.trace_r(u)
            if self.model.uhat_plan() is not None:             # disc.py:500-504
                uh, _ = self._eval(self.model.uhat_plan(),
                                   self._face_bind(d.fi_x, t, ul, ur, None, None, d.fi_n),
                                   d.fi_x.shape[:2], "uhat override")
            elif self.model.numflux.trace == "centered":
                uh = 0.5 * (ul + ur)
            else:
                uh = np.where(self.switch[:, None, None], ul, ur)
            vl = np.einsum("fq,fqi,fqj,fqa->faij", d.fi_wsj, ul - uh, d.fi_n,
                           d.fi_phi_l, optimize=True)
            vr = np.einsum("fq,fqi,fqj,fqa->faij", d.fi_wsj, ur - uh, d.fi_n,
                           d.fi_phi_r, optimize=True)
            scatter_add(rhs, self.topo.elem_l, vl)
            scatter_add(rhs, self.topo.elem_r, -vr)
        if self.topo.elem_b.shape[0]:
            ub = d.trace_b(u)
            uh = ub.copy()
            for tag, bc, idx in self.bc_groups:
                if bc.type == "dirichlet":
                    if homogeneous:
                        uh[idx] = 0.0
                    else:
                        g, _ = self._eval(self.model.bc_plan(tag),
                                          self._bind(d.fb_x[idx], t, n=d.fb_n[idx]),
                                          d.fb_x[idx].shape[:2], f"bc tag {tag}")
                        uh[idx] = g
            vb = np.einsum("fq,fqi,fqj,fqa->faij", d.fb_wsj, ub - uh, d.fb_n,
                           d.fb_phi, optimize=True)
            scatter_add(rhs, self.topo.elem_b, vb)
        return rhs

    # -- residual (disc.py:588-862) ------------------------------------------------
    def residual(self, u, t=0.0):
        return self._residual(u, t)

    def residual_tangent(self, u, du, t=0.0):
        return self._residual(u, t, du)

    def _residual(self, u, t, du=None):
        tan = du is not None
        d, m = self.d, self.master
        ne, nb = u.shape[:2]
        q = dq = None
        if self.kind == "D":
            q = self.compute_mixed(u, t)
            if tan:
                dq = self.compute_mixed(du, t, homogeneous=True)
        uq = np.einsum("qa,eai->eqi", m.phi, u)
        qq = None if q is None else np.einsum("qa,eaij->eqij", m.phi, q)
        seed = None
        if tan:
            duq = np.einsum("qa,eai->eqi", m.phi, du)
            dqq = None if dq is None else np.einsum("qa,eaij->eqij", m.phi, dq)
            seed = self._seed(duq, dqq)
        nq = m.phi.shape[0]
        bind = self._bind(d.xq, t, uq, qq)
        f, df = self._eval(self.model.flux_plan(), bind, (ne, nq), "flux", seed)
        s, ds = self._eval(self.model.source_plan(), bind, (ne, nq), "source", seed)
        if tan:
            f, s = df, ds
        f = f.reshape(ne, nq, self.ncu, self.nd)
        R = -np.einsum("eq,eqid,eqdr,qar->eai", d.wdetj, f, d.invjt, m.dphi,
                       optimize=True)
        R -= np.einsum("eq,eqi,qa->eai", d.wdetj, s, m.phi, optimize=True)
        if self.topo.elem_l.shape[0]:
            fh = self._interior_fhat(u, q, t, du, dq)
            vl = np.einsum("fq,fqi,fqa->fai", d.fi_wsj, fh, d.fi_phi_l, optimize=True)
            vr = np.einsum("fq,fqi,fqa->fai", d.fi_wsj, fh, d.fi_phi_r, optimize=True)
            scatter_add(R, self.topo.elem_l, vl)
            scatter_add(R, self.topo.elem_r, -vr)
        if self.topo.elem_b.shape[0]:
            fb = self._boundary_fhat(u, q, t, du, dq)
            vb = np.einsum("fq,fqi,fqa->fai", d.fb_wsj, fb, d.fb_phi, optimize=True)
            scatter_add(R, self.topo.elem_b, vb)
        return R

    def _tau_scale(self):
        flag = self.model.numflux.tau_over_h
        return self.kind == "D" if flag is None else bool(flag)

    def _interior_fhat(self, u, q, t, du, dq):
        """disc.py:657-751."""
        d = self.d
        tan = du is not None
        ul, ur = d.trace_l(u), d.trace_r(u)
        dul = dur = None
        if tan:
            dul, dur = d.trace_l(du), d.trace_r(du)
        shape = d.fi_x.shape[:2]
        sw = self.switch
        ql = qr = dql = dqr = None
        if q is not None:
            ql, qr = d.trace_l(q), d.trace_r(q)
            if tan:
                dql, dqr = d.trace_l(dq), d.trace_r(dq)
        fb = self._face_bind(d.fi_x, t, ul, ur, ql, qr, d.fi_n)
        fs = self._face_seed(dul, dur, dql, dqr) if tan else None
        if self.model.fhat_plan() is not None:                 # disc.py:753-758
            f, df = self._eval(self.model.fhat_plan(), fb, shape, "fhat override", fs)
            return df if tan else f
        if self.kind == "C":
            return self._llf(ul, ur, dul, dur, t, d.fi_x, d.fi_n, shape)
        if self.model.uhat_plan() is not None:                 # disc.py:500-504
            uh, duh = self._eval(self.model.uhat_plan(), fb, shape, "uhat override", fs)
        else:
            centered = self.model.numflux.trace == "centered"
            uh = 0.5 * (ul + ur) if centered else np.where(sw[:, None, None], ul, ur)
            duh = None
            if tan:
                duh = 0.5 * (dul + dur) if centered else np.where(sw[:, None, None], dul, dur)
        gc = self.model.numflux.grad_trace == "centered"
        qh = 0.5 * (ql + qr) if gc else np.where(sw[:, None, None, None], qr, ql)
        dqh = None
        if tan:
            dqh = 0.5 * (dql + dqr) if gc else np.where(sw[:, None, None, None], dqr, dql)
        bind = self._bind(d.fi_x, t, uh, qh, n=d.fi_n)
        f, df = self._eval(self.model.flux_plan(), bind, shape, "face flux",
                           self._seed(duh, dqh) if tan else None)
        fm = (df if tan else f).reshape(shape + (self.ncu, self.nd))
        fh = np.einsum("fqij,fqj->fqi", fm, d.fi_n)
        tau = float(self.model.numflux.tau)
        base = tau / d.fi_h[:, None, None] if self._tau_scale() else tau
        ws = self.model.wavespeed_plan()
        if ws is not None:
            ll, _ = self._eval(ws, self._bind(d.fi_x, t, u=ul, n=d.fi_n), shape, "wavespeed")
            lr, _ = self._eval(ws, self._bind(d.fi_x, t, u=ur, n=d.fi_n), shape, "wavespeed")
            base = base + np.maximum(ll, lr)
        return fh + base * ((dul - duh) if tan else (ul - uh))

    def _llf(self, ul, ur, dul, dur, t, x, n, shape):
        """disc.py:724-751."""
        tan = dul is not None
        fp, ws = self.model.flux_plan(), self.model.wavespeed_plan()
        fl, dfl = self._eval(fp, self._bind(x, t, ul, n=n), shape, "face flux",
                             self._seed(dul) if tan else None)
        fr, dfr = self._eval(fp, self._bind(x, t, ur, n=n), shape, "face flux",
                             self._seed(dur) if tan else None)
        ll, dll = self._eval(ws, self._bind(x, t, ul, n=n), shape, "wavespeed",
                             self._seed(dul) if tan else None)
        lr, dlr = self._eval(ws, self._bind(x, t, ur, n=n), shape, "wavespeed",
                             self._seed(dur) if tan else None)
        lam = np.maximum(ll, lr)
        sh = shape + (self.ncu, self.nd)
        if not tan:
            return 0.5 * np.einsum("fqij,fqj->fqi", fl.reshape(sh) + fr.reshape(sh), n) \
                + 0.5 * lam * (ul - ur)
        dfa = 0.5 * np.einsum("fqij,fqj->fqi", dfl.reshape(sh) + dfr.reshape(sh), n)
        dlam = np.where(ll >= lr, dll, dlr)
        return dfa + 0.5 * dlam * (ul - ur) + 0.5 * lam * (dul - dur)

    def _boundary_fhat(self, u, q, t, du, dq):
        """disc.py:762-862."""
        d = self.d
        tan = du is not None
        ub = d.trace_b(u)
        qb = None if q is None else d.trace_b(q)
        dub = d.trace_b(du) if tan else None
        dqb = d.trace_b(dq) if (tan and dq is not None) else None
        out = np.zeros(d.fb_x.shape[:2] + (self.ncu,))
        ws = self.model.wavespeed_plan()
        for tag, bc, idx in self.bc_groups:
            x, n = d.fb_x[idx], d.fb_n[idx]
            sh = x.shape[:2]
            g, _ = self._eval(self.model.bc_plan(tag), self._bind(x, t, n=n), sh,
                              f"bc tag {tag}")
            if bc.type == "neumann":
                if not tan:
                    out[idx] = g
                continue
            if self.kind == "C":
                fi, dfi = self._eval(self.model.flux_plan(), self._bind(x, t, ub[idx], n=n),
                                     sh, "boundary flux",
                                     self._seed(dub[idx]) if tan else None)
                fg, _ = self._eval(self.model.flux_plan(), self._bind(x, t, g, n=n), sh,
                                   "boundary flux")
                li, dli = self._eval(ws, self._bind(x, t, ub[idx], n=n), sh, "wavespeed",
                                     self._seed(dub[idx]) if tan else None)
                lg, _ = self._eval(ws, self._bind(x, t, g, n=n), sh, "wavespeed")
                lam = np.maximum(li, lg)
                s2 = sh + (self.ncu, self.nd)
                if not tan:
                    out[idx] = 0.5 * np.einsum("fqij,fqj->fqi", fi.reshape(s2) + fg.reshape(s2), n) \
                        + 0.5 * lam * (ub[idx] - g)
                else:
                    dl = np.where(li >= lg, dli, 0.0)
                    out[idx] = 0.5 * np.einsum("fqij,fqj->fqi", dfi.reshape(s2), n) \
                        + 0.5 * dl * (ub[idx] - g) + 0.5 * lam * dub[idx]
                continue
            seed = self._seed(np.zeros_like(dub[idx]),
                              None if dqb is None else dqb[idx]) if tan else None
            f, df = self._eval(self.model.flux_plan(),
                               self._bind(x, t, g, None if qb is None else qb[idx], n=n),
                               sh, "boundary flux", seed)
            fn = np.einsum("fqij,fqj->fqi", (df if tan else f).reshape(sh + (self.ncu, self.nd)), n)
            tau = float(self.model.numflux.tau)
            tau = tau / d.fb_h[idx][:, None, None] if self._tau_scale() else tau
            if ws is not None:
                li, _ = self._eval(ws, self._bind(x, t, u=ub[idx], n=n), sh, "wavespeed")
                lg, _ = self._eval(ws, self._bind(x, t, u=g, n=n), sh, "wavespeed")
                tau = tau + np.maximum(li, lg)
            out[idx] = fn + tau * (dub[idx] if tan else (ub[idx] - g))
        return out

    # -- mass (disc.py:897-948) -------------------------------------------------------
    def mass_apply(self, u, vu, t=0.0):
        d, phi = self.d, self.master.phi
        if self.mass_const:
            mv, _ = self._eval(self.model.mass_plan(), {"t": 0.0}, (1, 1), "mass")
            mq = np.broadcast_to(mv.reshape(1, 1, self.ncu), d.xq.shape[:2] + (self.ncu,))
        else:
            uq = np.einsum("qa,eai->eqi", phi, u)
            mq, _ = self._eval(self.model.mass_plan(), self._bind(d.xq, t, uq),
                               d.xq.shape[:2], "mass")
        vq = np.einsum("qa,eai->eqi", phi, vu)
        return np.einsum("eq,eqi,qa->eai", d.wdetj, mq * vq, phi, optimize=True)

    def mass_tangent_extra(self, u, y, du, t=0.0):
        """disc.py:927-948: (dm/du . du) y, None for a constant mass."""
        if self.mass_const:
            return None
        d, phi = self.d, self.master.phi
        uq = np.einsum("qa,eai->eqi", phi, u)
        duq = np.einsum("qa,eai->eqi", phi, du)
        _, dm = self._eval(self.model.mass_plan(), self._bind(d.xq, t, uq),
                           d.xq.shape[:2], "mass", self._seed(duq))
        yq = np.einsum("qa,eai->eqi", phi, y)
        return np.einsum("eq,eqi,qa->eai", d.wdetj, dm * yq, phi, optimize=True)
