"""Host table builder: (model, mesh, topology, master) -> device tables.

Replaces the reference's dense per-quadrature-point ``Discretization``
(disc.py:74-239, ~1.9 KB/DOF at hex p=3) with what the B200 kernels read:

* per element: detJ and invJ^T (affine elements, 80 B);
* per element-face: neighbour element (or boundary row), an info word
  (interior/dirichlet/neumann, left/right side, the reference's switch bit,
  the neighbour node-map id) and the penalty tau;
* a handful of neighbour node maps (own face node -> neighbour volume node,
  found by matching physical node coordinates, periodic shift applied);
* 1D GLL operators D1, M1, S1 and the lift columns M1^-1 e_0, M1^-1 e_p;
* flux coefficients of a flux that is linear in (u, q).

The switch bits are computed with the reference's own floating-point
pipeline (disc.py:139-180, 285-287) because on simplices and on faces with
n . beta_hat = 0 they are decided by rounding; the tests pin them against the
reference bit for bit.  Everything else is exact-arithmetic geometry.
"""

from __future__ import annotations

import numpy as np

from . import refelem
from .expr import evaluate
from .refelem import FACES, face_map

# local face -> (normal axis, high side) for the tensor kinds
FACE_AXIS = {"line": [(0, 0), (0, 1)],
             "quad": [(1, 0), (0, 1), (1, 1), (0, 0)],
             "hex": [(2, 0), (2, 1), (1, 0), (1, 1), (0, 0), (0, 1)]}


class DiscError(ValueError):
    pass


class KernelNanError(DiscError):
    pass


# ---------------------------------------------------------------------------
# plan analysis
# ---------------------------------------------------------------------------


def affine_form(plan, mu, variables):
    """Symbolic affine forms of a plan's outputs in `variables` with
    constant coefficients (mu substituted).  Returns a list of
    (coeffs: dict var->float, const: float) or None if any output is not
    affine with constant coefficients."""
    forms = []
    for ins in plan.instructions:
        tag = ins[0]
        f = None
        if tag == "const":
            f = ({}, float(ins[1]))
        elif tag == "sym":
            s = ins[1]
            if s in variables:
                f = ({s: 1.0}, 0.0)
            elif s in mu:
                f = ({}, float(mu[s]))
        elif tag == "neg":
            a = forms[ins[1]]
            if a is not None:
                f = ({k: -v for k, v in a[0].items()}, -a[1])
        elif tag in ("add", "sub"):
            a, b = forms[ins[1]], forms[ins[2]]
            if a is not None and b is not None:
                s = 1.0 if tag == "add" else -1.0
                co = dict(a[0])
                for k, v in b[0].items():
                    co[k] = co.get(k, 0.0) + s * v
                f = (co, a[1] + s * b[1])
        elif tag == "mul":
            a, b = forms[ins[1]], forms[ins[2]]
            if a is not None and b is not None:
                if not a[0]:
                    f = ({k: a[1] * v for k, v in b[0].items()}, a[1] * b[1])
                elif not b[0]:
                    f = ({k: b[1] * v for k, v in a[0].items()}, a[1] * b[1])
        elif tag == "div":
            a, b = forms[ins[1]], forms[ins[2]]
            if a is not None and b is not None and not b[0] and b[1] != 0.0:
                f = ({k: v / b[1] for k, v in a[0].items()}, a[1] / b[1])
        elif tag in ("call", "pow"):
            args = ins[2] if tag == "call" else (ins[1], ins[2])
            fa = [forms[x] for x in args]
            if all(x is not None and not x[0] for x in fa):
                vals = [np.array([x[1]]) for x in fa]
                from .expr import _binop, _fn
                with np.errstate(all="ignore"):
                    v = _fn(ins[1], vals) if tag == "call" else _binop("pow", *vals)
                f = ({}, float(v[0]))
        forms.append(f)
    out = []
    for r in plan.outputs:
        if forms[r] is None:
            return None
        out.append(forms[r])
    return out


def uses_any(plan, prefixes):
    return any(s.startswith(prefixes) for s in
               {i[1] for i in plan.instructions if i[0] == "sym"})


def plan_is_zero(plan):
    return all(plan.instructions[r] == ("const", 0.0) for r in plan.outputs)


# ---------------------------------------------------------------------------
# reference-faithful switch bits (disc.py:139-180, 285-287)
# ---------------------------------------------------------------------------


def reference_switch(mesh, topo, master, geom, chunk=1 << 16):
    nd = mesh.nd
    nfi = topo.elem_l.shape[0]
    nbar = np.zeros((nfi, nd))
    for lf in range(master.n_faces):
        sel = np.nonzero(topo.face_l == lf)[0]
        if sel.size == 0:
            continue
        gd = geom.eval_basis_grad(master.faces[lf].xi)
        _, T = face_map(mesh.elem_kind, lf)
        for c0 in range(0, sel.size, chunk):
            s = sel[c0:c0 + chunk]
            ho = mesh.ho_nodes[topo.elem_l[s]]
            if nd == 1:
                raise DiscError("1D meshes are not supported by the B200 path")
            nbar[s] = _face_nbar(gd, T, ho)
    beta = np.ones(nd) / np.sqrt(nd)
    return (nbar @ beta) > 0.0


def _tangents(gd, T, ho, rows=4096):
    """np.einsum("qgd,sd,kgc->kqcs", gd, T, ho) -- the reference's own
    face-tangent contraction, whose rounding decides the switch bit of
    near-tie faces -- split over element rows on host threads (numpy's
    einsum releases the GIL).  Every output row is the same einsum on the
    same operands, so the result is bit-identical to the single call."""
    k = ho.shape[0]
    if k <= rows:
        return np.einsum("qgd,sd,kgc->kqcs", gd, T, ho)
    from concurrent.futures import ThreadPoolExecutor
    import os
    out = np.empty((k, gd.shape[0], ho.shape[2], T.shape[0]))
    starts = range(0, k, rows)
    # the einsum's own evaluation order, restated as broadcast array ops (~10x
    # faster than the 3-operand einsum loop): per geometry node g a partial
    # sum over d of (gd T) ho, the partials added in g order.  Used only when
    # it reproduces the einsum bit for bit on the first row block.
    out[:rows] = np.einsum("qgd,sd,kgc->kqcs", gd, T, ho[:rows])
    fast = np.array_equal(_tangents_ordered(gd, T, ho[:rows]), out[:rows])

    def run(a):
        if a == 0:
            return
        if fast:
            out[a:a + rows] = _tangents_ordered(gd, T, ho[a:a + rows])
        else:
            out[a:a + rows] = np.einsum("qgd,sd,kgc->kqcs", gd, T, ho[a:a + rows])

    with ThreadPoolExecutor(max(1, min(32, os.cpu_count() or 1))) as ex:
        list(ex.map(run, starts))
    return out


def _tangents_ordered(gd, T, ho):
    nq, ng, nrd = gd.shape
    out = np.zeros((ho.shape[0], nq, ho.shape[2], T.shape[0]))
    for g in range(ng):
        part = np.zeros_like(out)
        for d in range(nrd):
            c = gd[:, g, d][:, None] * T[:, d][None, :]                 # (q, s)
            part += c[None, :, None, :] * ho[:, g, :][:, None, :, None]
        out += part
    return out


def _face_nbar_numpy(gd, T, ho):
    nd = ho.shape[2]
    tang = _tangents(gd, T, ho)
    if nd == 2:
        t = tang[:, :, :, 0]
        nv = np.stack([t[:, :, 1], -t[:, :, 0]], axis=-1)
    else:
        nv = np.cross(tang[:, :, :, 0], tang[:, :, :, 1])
    mag = np.linalg.norm(nv, axis=-1)
    n = np.zeros((ho.shape[0], gd.shape[0], nd))
    n[:] = nv / mag[:, :, None]
    return n.mean(axis=1)


def _face_nbar(gd, T, ho, check=256):
    """Mean unit face normal in the reference's operation order
    (disc.py:167-178, 122): the native ldg_face_nbar (host C++, OpenMP) when
    the library is present and reproduces the numpy pipeline bit for bit on
    the first faces, else the numpy pipeline itself."""
    k, nd = ho.shape[0], ho.shape[2]
    if k == 0 or nd not in (2, 3):
        return _face_nbar_numpy(gd, T, ho)
    try:
        from . import _lib
        lib = _lib.load(require_gpu=False)
    except Exception:                                   # setup needs no GPU
        return _face_nbar_numpy(gd, T, ho)
    import ctypes as C
    gd_, T_, ho_ = (np.ascontiguousarray(a, dtype=np.float64) for a in (gd, T, ho))
    out = np.empty((k, nd))
    rc = lib.ldg_face_nbar(k, gd_.shape[0], gd_.shape[1], gd_.shape[2], nd,
                           gd_.ctypes.data_as(C.c_void_p), T_.ctypes.data_as(C.c_void_p),
                           ho_.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p))
    if rc != 0 or not np.array_equal(out[:check], _face_nbar_numpy(gd, T, ho[:check])):
        return _face_nbar_numpy(gd, T, ho)
    return out


def _reference_switch_subset(mesh, master, geom, elems, lfs):
    """reference_switch restricted to the given (left element, face) list."""
    nd = mesh.nd
    out = np.zeros(elems.size, dtype=bool)
    nbar = np.zeros((elems.size, nd))
    for lf in np.unique(lfs):
        sel = np.nonzero(lfs == lf)[0]
        gd = geom.eval_basis_grad(master.faces[lf].xi)
        _, T = face_map(mesh.elem_kind, lf)
        nbar[sel] = _face_nbar(gd, T, mesh.ho_nodes[elems[sel]])
    beta = np.ones(nd) / np.sqrt(nd)
    out[:] = (nbar @ beta) > 0.0
    return out


# ---------------------------------------------------------------------------
# table builder
# ---------------------------------------------------------------------------


def _line_master_tables(m):
    """1D GLL / Gauss tables of a line master in the attributes the tensor
    tables read (a line master's own tabulations are already 1D)."""
    if getattr(m, "phi1d", None) is None:
        m.nodes1d = np.asarray(m.nodes)[:, 0].copy()
        m.phi1d = np.asarray(m.phi)
        m.dphi1d = np.asarray(m.dphi)[:, :, 0]
        m.quad1d = (np.asarray(m.quad_pts)[:, 0].copy(), np.asarray(m.quad_wts))


def mesh_is_affine(mesh):
    """True when every element's geometry map is affine (the Jacobian at the
    reference corners agrees to roundoff) -- the fused / dense kernels'
    precondition; curved meshes run on the generated path."""
    geom = refelem.build_geom_master(mesh.elem_kind, mesh.p_geom)
    gd = geom.eval_basis_grad(refelem.VERTS[mesh.elem_kind])
    J = np.einsum("egd,vgr->evdr", mesh.ho_nodes, gd)
    return not bool(np.max(np.abs(J - J[:, :1])) > 1e-11 * max(mesh.diameter(), 1.0))


class TensorTables:
    """Host arrays for the tensor-product (quad/hex) kernels."""

    def __init__(self, model, mesh, topo, master, nonlinear=False):
        """`nonlinear`: tables for the generated-kernel path (nonlinear.py):
        any kind C / D model, the state-dependent penalty evaluated on the
        device; otherwise the linear constant-coefficient fused path."""
        self.model, self.mesh, self.topo, self.master = model, mesh, topo, master
        self.nonlinear = nonlinear
        kind = master.kind
        if kind != mesh.elem_kind:
            raise DiscError("master element kind does not match the mesh")
        if kind not in ("quad", "hex") and not (kind == "line" and nonlinear):
            raise DiscError(f"B200 tensor path needs quad/hex elements, got {kind}")
        if kind == "line":
            _line_master_tables(master)
        if model.kind not in (("C", "D", "W") if nonlinear else ("D",)):
            raise DiscError(f"B200 path supports kind C/D/W models, got {model.kind}"
                            if nonlinear else
                            f"linear B200 path supports kind D models, got {model.kind}")
        if not nonlinear and (model.nw > 0 or model.numflux.uhat is not None or
                              model.numflux.fhat is not None):
            raise DiscError("ODE blocks and u^/f^ overrides run on the generated path")
        self.nd, self.p, self.ncu = mesh.nd, master.p, model.ncu
        self.n1 = master.p + 1
        if self.n1 > 7 or self.ncu > (5 if nonlinear else 3):
            raise DiscError("tensor path supports p <= 6 and ncu <= 3 (5 on the generated path)")
        if master.quad_degree < 2 * master.p:
            raise DiscError("tensor path needs quadrature degree >= 2p (exact mass/stiffness)")
        self.nf = 2 * self.nd
        self.nfn = self.n1 ** (self.nd - 1)
        self.ne = mesh.connectivity.shape[0]
        self._check_gll()
        self._operators()
        self._geometry()
        if nonlinear:
            self.flux_uses_u = True
            self.source_zero = plan_is_zero(model.source_plan())
        else:
            self._flux_coefficients()
        self._faces()

    # -- reference element -----------------------------------------------------
    def _check_gll(self):
        m = self.master
        x1 = refelem.gauss_lobatto(m.p)
        if m.nodes1d is None or np.max(np.abs(m.nodes1d - x1)) > 1e-13:
            raise DiscError("tensor path needs GLL solution nodes")
        L = m.phi1d
        if self.nd == 1:
            kron = L
        elif self.nd == 3:
            kron = np.einsum("zk,yj,xi->zyxkji", L, L, L).reshape(m.phi.shape)
        else:
            kron = np.einsum("yj,xi->yxji", L, L).reshape(m.phi.shape)
        if np.max(np.abs(kron - m.phi)) > 1e-12:
            raise DiscError("master basis is not the tensor GLL basis")

    def _operators(self):
        m = self.master
        n1 = self.n1
        L, dL = m.phi1d, m.dphi1d
        w = m.quad1d[1]
        basis = refelem.TensorLegendreBasis(1, m.p)
        V = basis.eval(m.nodes1d[:, None])
        Vd = basis.grad(m.nodes1d[:, None])[:, :, 0]
        self.d1 = Vd @ np.linalg.inv(V)                       # D[i][m] = l'_m(x_i)
        self.m1 = np.einsum("q,qa,qb->ab", w, L, L)
        self.s1 = np.einsum("q,qa,qb->ab", w, dL, L)          # S[a][b] = int l'_a l_b
        mi = np.linalg.inv(self.m1)
        self.clo = mi[:, 0].copy()
        self.chi = mi[:, n1 - 1].copy()
        self.m1inv = mi

    def _geometry(self):
        mesh, nd = self.mesh, self.nd
        geom = refelem.build_geom_master(mesh.elem_kind, mesh.p_geom)
        self.geom_master = geom
        corners = refelem.VERTS[mesh.elem_kind]
        gd = geom.eval_basis_grad(corners)                    # (nv, ng, nd)
        J = np.einsum("egd,vgr->evdr", mesh.ho_nodes, gd)
        scale = max(mesh.diameter(), 1.0)
        self.curved = bool(np.max(np.abs(J - J[:, :1])) > 1e-11 * scale)
        if self.curved:
            if not self.nonlinear:
                raise DiscError("curved (non-affine) elements run on the generated path "
                                "(quad / hex) only")
            self._curved_geometry(geom)
            # element-level affine stand-ins (the Jacobian at the reference
            # centre): only the table builders' approximate uses read them
            J = np.einsum("egd,gr->edr", mesh.ho_nodes,
                          geom.eval_basis_grad(np.zeros((1, nd)))[0])
        else:
            J = J[:, 0]
        # numpy's det / inv as the reference calls them (disc.py:94-96): the
        # geometry bits feed every operator coefficient, and the 1e-10
        # solution bar of the identity-preconditioned solves rides on them
        self.detj = np.linalg.det(J)
        if np.any(self.detj <= 0):
            bad = int(np.argmax(self.detj <= 0))
            raise DiscError(f"nonpositive Jacobian in element {bad}")
        self.invjt = np.linalg.inv(J).transpose(0, 2, 1)
        self.x0 = np.einsum("egd,g->ed", mesh.ho_nodes,
                            geom.eval_basis(np.zeros((1, nd)))[0])  # image of xi = 0
        self.J = J
        self.geo = np.concatenate([self.detj[:, None], self.invjt.reshape(self.ne, -1)], axis=1)
        m = self.master
        self.elem_vol = self.wdetj_q.sum(axis=1) if self.curved else self.detj * m.quad_wts.sum()

    def _curved_geometry(self, geom):
        """Per-quadrature-point metrics of non-affine elements, the
        reference's own pipeline (disc.py:91-104): J = sum_g x_g grad N_g at
        the volume points, detJ, invJ^T, the weighted detJ and the physical
        points; per-face-point normals / weighted surface jacobians follow
        in face_point_geometry (disc.py:139-180)."""
        mesh, m = self.mesh, self.master
        ho = mesh.ho_nodes
        gphi = geom.eval_basis(m.quad_pts)
        gdphi = geom.eval_basis_grad(m.quad_pts)
        Jq = np.einsum("egd,qgr->eqdr", ho, gdphi)
        detj = np.linalg.det(Jq)
        if np.any(detj <= 0):
            bad = int(np.argwhere(detj.min(axis=1) <= 0)[0][0])
            raise DiscError(f"nonpositive Jacobian in element {bad}")
        self.detj_q = detj
        self.invjt_q = np.linalg.inv(Jq).transpose(0, 1, 3, 2)
        self.wdetj_q = m.quad_wts[None, :] * detj
        self.xq_q = np.einsum("qg,egd->eqd", gphi, ho)

    def face_point_geometry(self, elems, lf, xi=None):
        """(x, unit normal, |t1 x t2| without the weight) at reference face
        points xi (default: the master's face rule) of local face lf -- the
        reference's face pipeline (disc.py:139-180: tangents
        dx/dsigma = grad N . T, n = t1 x t2 / |t1 x t2|)."""
        geom = self.geom_master
        xi = self.master.faces[lf].xi if xi is None else xi
        ho = self.mesh.ho_nodes[elems]
        x = np.einsum("qg,kgd->kqd", geom.eval_basis(xi), ho)
        _, T = face_map(self.master.kind, lf)
        tang = _tangents(geom.eval_basis_grad(xi), T, ho)
        if self.nd == 2:
            t = tang[:, :, :, 0]
            nv = np.stack([t[:, :, 1], -t[:, :, 0]], axis=-1)
        else:
            nv = np.cross(tang[:, :, :, 0], tang[:, :, :, 1])
        mag = np.linalg.norm(nv, axis=-1)
        return x, nv / mag[:, :, None], mag

    def node_coords(self, elems=None, nodes=None):
        """Physical coordinates of solution nodes (the geometry map; affine:
        x0 + J xi)."""
        m = self.master
        xi = m.nodes if nodes is None else m.nodes[nodes]
        e = slice(None) if elems is None else elems
        if getattr(self, "curved", False):
            ho = self.mesh.ho_nodes[e]
            return np.einsum("ng,egd->end", self.geom_master.eval_basis(xi), ho)
        return self.x0[e][:, None, :] + np.einsum("edr,nr->end", self.J[e], xi)

    def _flux_coefficients(self):
        model, nd, ncu = self.model, self.nd, self.ncu
        mu = model.mu_bindings()
        var = [f"u{i + 1}" for i in range(ncu)] + \
            [f"q{i + 1}_{j + 1}" for i in range(ncu) for j in range(nd)]
        forms = affine_form(model.flux_plan(), mu, set(var))
        if forms is None:
            raise DiscError("B200 path needs a flux linear in (u, q) with constant "
                            "coefficients (nonlinear fluxes are not supported yet)")
        if any(abs(c) > 0 for _, c in forms):
            raise DiscError("flux has a state-independent part; not supported")
        self.au = np.zeros((5, 3, 5))
        self.aq = np.zeros((5, 3, 5, 3))
        for c in range(ncu):
            for d in range(nd):
                co = forms[c * nd + d][0]
                for k in range(ncu):
                    self.au[c, d, k] = co.get(f"u{k + 1}", 0.0)
                    for e in range(nd):
                        self.aq[c, d, k, e] = co.get(f"q{k + 1}_{e + 1}", 0.0)
        self.flux_uses_u = bool(np.any(self.au != 0))
        if uses_any(model.source_plan(), ("u", "q", "w")):
            raise DiscError("state-dependent sources are not supported on the B200 path yet")
        self.source_zero = plan_is_zero(model.source_plan())
        mp = model.mass_plan()
        mforms = affine_form(mp, mu, set())
        self.mass_const = mforms is not None
        self.mass_coef = np.zeros(5)
        if mforms is not None:
            for c in range(ncu):
                self.mass_coef[c] = mforms[c][1]
        ws = model.wavespeed_plan()
        if ws is not None and uses_any(ws, ("u", "q", "w", "x")):
            raise DiscError("wavespeed depending on the state or x is not supported yet")

    # -- faces -------------------------------------------------------------------
    def face_node_vol(self, lf):
        """Volume node index of each face node t (increasing volume order)."""
        n1, nd = self.n1, self.nd
        ax, hi = FACE_AXIS[self.master.kind][lf]
        io = n1 - 1 if hi else 0
        t = np.arange(self.nfn)
        if nd == 1:
            return np.full(1, io)
        if nd == 2:
            return io + n1 * t if ax == 0 else t + n1 * io
        a, b = t % n1, t // n1
        if ax == 0:
            return io + n1 * a + n1 * n1 * b
        if ax == 1:
            return a + n1 * io + n1 * n1 * b
        return a + n1 * b + n1 * n1 * io

    def face_normal_area(self, elems, lf):
        """Outward unit normal and |t1 x t2| of local face lf (affine; for
        curved elements the face-rule average normal and the area over the
        reference face measure, for the per-face quantities only)."""
        if self.nd == 1:
            # a point face: the reference normal, unit measure (disc.py:158-163)
            sgn = 1.0 if FACE_AXIS[self.master.kind][lf][1] else -1.0
            elems = np.asarray(elems)
            return np.full((elems.size, 1), sgn), np.ones(elems.size)
        if getattr(self, "curved", False):
            _, n, mag = self.face_point_geometry(elems, lf)
            w = self.master.faces[lf].weights
            nb = n.mean(axis=1)
            return nb / np.linalg.norm(nb, axis=1)[:, None], (mag * w).sum(axis=1) / w.sum()
        _, T = face_map(self.master.kind, lf)
        tn = np.cross(T[0], T[1]) if self.nd == 3 else np.array([T[0][1], -T[0][0]])
        v = np.einsum("edr,r->ed", self.invjt[elems], tn)
        ln = np.linalg.norm(v, axis=1)
        return v / ln[:, None], self.detj[elems] * ln

    def _faces(self):
        topo, model, mesh = self.topo, self.model, self.mesh
        ne, nf, nfn = self.ne, self.nf, self.nfn
        fnbr = np.full((ne, nf), -1, dtype=np.int32)
        finfo = np.full((ne, nf), -1, dtype=np.int32)
        ftau = np.zeros((ne, nf))
        nfi = topo.elem_l.shape[0]
        el, fl, er, fr = (np.asarray(a, dtype=np.int64) for a in
                          (topo.elem_l, topo.face_l, topo.elem_r, topo.face_r))
        # switch bits, the reference way
        self.switch = self._switch_bits(el, fl)
        # penalty
        tau = float(model.numflux.tau)
        over_h = model.numflux.tau_over_h
        over_h = (model.kind == "D") if over_h is None else bool(over_h)   # disc.py:701-705
        fw = self.master.faces[0].weights.sum()
        ws = model.wavespeed_plan()
        mu = model.mu_bindings()

        def lam(normals):
            # constant wavespeed folded into tau (linear path); the generated
            # path evaluates lambda(u) per face point on the device
            if ws is None or normals.shape[0] == 0 or self.nonlinear:
                return 0.0
            b = {"t": 0.0, **mu}
            for k in range(self.nd):
                b[f"n{k + 1}"] = normals[:, k]
            return evaluate(ws, b)[0]

        n_l = np.zeros((nfi, self.nd))
        area = np.zeros(nfi)
        for lf in range(nf):
            sel = np.nonzero(fl == lf)[0]
            if sel.size:
                n_l[sel], sj = self.face_normal_area(el[sel], lf)
                area[sel] = sj * fw
        fi_h = 0.5 * (self.elem_vol[el] + self.elem_vol[er]) / np.maximum(area, 1e-300)
        if self.nd == 1:                                   # disc.py:130-133
            fi_h = 0.5 * (self.elem_vol[el] + self.elem_vol[er])
        tau_i = (tau / fi_h if over_h else np.full(nfi, tau)) + lam(n_l)
        self.fi_h = fi_h
        # neighbour node maps
        maps, mapid_l, mapid_r = self._node_maps(el, fl, er, fr)
        self.nmap = maps
        sw = self.switch.astype(np.int32)
        fnbr[el, fl] = er
        fnbr[er, fr] = el
        finfo[el, fl] = 0 | (sw << 3) | (fr.astype(np.int32) << 4) | (mapid_l << 8)
        finfo[er, fr] = 0 | 4 | (sw << 3) | (fl.astype(np.int32) << 4) | (mapid_r << 8)
        ftau[el, fl] = tau_i
        ftau[er, fr] = tau_i
        # boundary faces
        eb, fb, tb = (np.asarray(a, dtype=np.int64) for a in
                      (topo.elem_b, topo.face_b, topo.tag_b))
        self.bc_groups = []
        for tag in (np.unique(tb) if tb.size else []):
            tag = int(tag)
            if tag not in model.bcs:
                raise DiscError(f"mesh boundary tag {tag} has no [bc] entry")
            bc = model.bcs[tag]
            if bc.type == "periodic":
                raise DiscError(f"tag {tag} is periodic in the model but was not "
                                "paired in the mesh topology")
            if bc.type == "absorbing" and model.kind != "W":
                raise DiscError("absorbing boundaries require a wave model")   # disc.py:300-301
            if bc.type not in ("dirichlet", "neumann") and not (
                    self.nonlinear and bc.type == "absorbing"):
                raise DiscError(f"boundary type {bc.type!r} is not supported on the B200 path")
            self.bc_groups.append((tag, bc, np.nonzero(tb == tag)[0]))
        kinds = np.zeros(eb.size, dtype=np.int32)
        for tag, bc, idx in self.bc_groups:
            kinds[idx] = {"dirichlet": 1, "neumann": 2, "absorbing": 3}[bc.type]
        nb_ = np.zeros((eb.size, self.nd))
        area_b = np.zeros(eb.size)
        for lf in range(nf):
            sel = np.nonzero(fb == lf)[0]
            if sel.size:
                nb_[sel], sj = self.face_normal_area(eb[sel], lf)
                area_b[sel] = sj * fw
        fb_h = self.elem_vol[eb] / np.maximum(area_b, 1e-300)
        if self.nd == 1:
            fb_h = self.elem_vol[eb]
        tau_b = (tau / fb_h if over_h else np.full(eb.size, tau)) + lam(nb_)
        self.fb_h = fb_h
        self.n_left, self.sj_left, self.n_bnd, self.sj_bnd = n_l, area / fw, nb_, area_b / fw
        self.tau_i, self.tau_b = tau_i, tau_b
        fnbr[eb, fb] = np.arange(eb.size, dtype=np.int32)
        finfo[eb, fb] = kinds
        ftau[eb, fb] = tau_b
        if np.any(finfo < 0):
            e = int(np.argwhere(finfo < 0)[0][0])
            raise DiscError(f"element {e} has an unclassified face")
        self.fnbr, self.finfo, self.ftau = fnbr, finfo, ftau
        self.n_boundary = eb.size
        self.eb, self.fb = eb, fb

    def _switch_bits(self, el, fl):
        """n_bar . beta_hat > 0 (disc.py:285-287).  Faces whose affine normal
        is clearly off the n.beta = 0 plane take the sign directly; near-tie
        faces are recomputed with the reference pipeline so rounding decides
        them exactly as it does in the reference."""
        nfi = el.size
        if nfi == 0:
            return np.zeros(0, dtype=bool)
        if self.nd == 1:
            # nbar = the reference face normal (disc.py:158-163), beta_hat = 1
            return np.asarray(fl) == 1
        if getattr(self, "curved", False):
            # non-affine faces: the reference's own normal-average pipeline
            return _reference_switch_subset(self.mesh, self.master, self.geom_master, el, fl)
        n = np.zeros((nfi, self.nd))
        for lf in range(self.nf):
            sel = np.nonzero(fl == lf)[0]
            if sel.size:
                n[sel], _ = self.face_normal_area(el[sel], lf)
        d = n @ (np.ones(self.nd) / np.sqrt(self.nd))
        sw = d > 0.0
        near = np.abs(d) < 1e-8
        if near.any():
            idx = np.nonzero(near)[0]
            sw[idx] = _reference_switch_subset(self.mesh, self.master, self.geom_master,
                                               el[idx], fl[idx])
        return sw

    def _node_maps(self, el, fl, er, fr, chunk=1 << 15):
        """Own face node t -> neighbour volume node, both sides; returns
        (unique maps, map id of the left side, map id of the right side).

        Per (face_l, face_r) class a candidate permutation is found by
        nearest-node matching on one face and verified on all faces of the
        class at once; faces it does not fit (other orientations) go round
        again, so structured meshes cost one vectorised check per class."""
        nfi, nfn = el.size, self.nfn
        if nfi == 0:
            return np.zeros((1, nfn), dtype=np.int32), np.zeros(0, np.int32), np.zeros(0, np.int32)
        perm_lr = np.zeros((nfi, nfn), dtype=np.int64)   # left t -> right t'
        tr = np.asarray(self.topo.translation, dtype=float)
        if tr.shape[0] != nfi:
            tr = np.zeros((nfi, self.nd))
        tol2 = (1e-9 * max(self.mesh.diameter(), 1.0)) ** 2
        for a in range(self.nf):
            va = self.face_node_vol(a)
            for b in range(self.nf):
                rem = np.nonzero((fl == a) & (fr == b))[0]
                vb = self.face_node_vol(b)
                while rem.size:
                    f0 = rem[:1]
                    xl = self.node_coords(el[f0], va) + tr[f0][:, None, :]
                    xr = self.node_coords(er[f0], vb)
                    d2 = np.sum((xl[:, :, None, :] - xr[:, None, :, :]) ** 2, axis=3)
                    p = np.argmin(d2[0], axis=1)
                    if d2[0][np.arange(nfn), p].max() > tol2 or \
                            np.unique(p).size != nfn:
                        raise DiscError("non-conforming face nodes (hanging or "
                                        "misaligned faces are not supported)")
                    ok = np.zeros(rem.size, dtype=bool)
                    for c0 in range(0, rem.size, chunk):
                        s_ = rem[c0:c0 + chunk]
                        xl = self.node_coords(el[s_], va) + tr[s_][:, None, :]
                        xr = self.node_coords(er[s_], vb[p])
                        ok[c0:c0 + chunk] = np.sum((xl - xr) ** 2, axis=2).max(axis=1) <= tol2
                    perm_lr[rem[ok]] = p
                    rem = rem[~ok]
        vol = np.stack([self.face_node_vol(a) for a in range(self.nf)])   # (nf, nfn)
        map_l = vol[fr[:, None], perm_lr]                   # left t -> right vol node
        inv = np.argsort(perm_lr, axis=1)                   # right t' -> left t
        map_r = vol[fl[:, None], inv]
        # distinct maps via a hash of (class, permutation) rows
        allm = np.concatenate([map_l, map_r], axis=0)
        key = allm @ (np.int64(self.n1 ** self.nd + 1) ** np.arange(nfn, dtype=np.int64) %
                      np.int64(2 ** 61 - 1))
        _, first, ids = np.unique(key, return_index=True, return_inverse=True)
        uniq = allm[first]
        if not np.array_equal(uniq[ids], allm):
            raise DiscError("face node map hashing collided")
        ids = ids.reshape(-1).astype(np.int32)
        if uniq.shape[0] >= (1 << 16):
            raise DiscError("too many distinct face orientations")
        return uniq.astype(np.int32), ids[:nfi], ids[nfi:]

    # -- time-dependent data ---------------------------------------------------------
    def boundary_projection(self, t):
        """(n_bfaces, nfn, ncu) L2 projection of Dirichlet / Neumann data onto
        the face nodes: the face quadrature of any trace against it equals the
        reference's quadrature of the raw data (disc.py:559-563, 775-782)."""
        nb_ = self.n_boundary
        out = np.zeros((nb_, self.nfn, self.ncu))
        if nb_ == 0:
            return out
        m, geom, model = self.master, self.geom_master, self.model
        mu = model.mu_bindings()
        w = m.faces[0].weights
        for tag, bc, idx in self.bc_groups:
            if bc.type == "absorbing":
                continue
            plan = model.bc_plan(tag)
            for lf in range(self.nf):
                s = idx[self.fb[idx] == lf]
                if s.size == 0:
                    continue
                face = m.faces[lf]
                xq = np.einsum("qg,kgd->kqd", geom.eval_basis(face.xi),
                               self.mesh.ho_nodes[self.eb[s]])
                n, _ = self.face_normal_area(self.eb[s], lf)
                b = {"t": float(t), **mu}
                for k in range(self.nd):
                    b[f"x{k + 1}"] = xq[..., k].ravel()
                    b[f"n{k + 1}"] = np.repeat(n[:, k], xq.shape[1])
                g = evaluate(plan, b)                       # (ncu, B)
                if g.shape[1] != xq.shape[0] * xq.shape[1]:
                    g = np.broadcast_to(g, (g.shape[0], xq.shape[0] * xq.shape[1]))
                if not np.isfinite(g).all():
                    col = int(np.argwhere(~np.isfinite(g))[0][1])
                    raise KernelNanError(f"bc tag {tag} kernel produced non-finite "
                                         f"values (first at element {col // xq.shape[1]})")
                g = g.reshape(self.ncu, s.size, -1).transpose(1, 2, 0)   # (k, nqf, ncu)
                Phi = face.phi[:, self.face_node_vol(lf)]              # (nqf, nfn)
                Mf = Phi.T @ (w[:, None] * Phi)
                P = np.linalg.solve(Mf, Phi.T * w[None, :])            # (nfn, nqf)
                out[s] = np.einsum("tq,kqc->ktc", P, g)
        return out

    def source_load(self, t):
        """(ne, nb, ncu) = -int s(x, t) phi (disc.py:621-629), or None."""
        if self.source_zero:
            return None
        m, model = self.master, self.model
        b = {"t": float(t), **model.mu_bindings()}
        out = np.empty((self.ne, m.n_nodes, self.ncu))
        step = 1 << 15
        for c0 in range(0, self.ne, step):
            e = np.arange(c0, min(self.ne, c0 + step))
            xq = self.x0[e][:, None, :] + np.einsum("edr,qr->eqd", self.J[e], m.quad_pts)
            for k in range(self.nd):
                b[f"x{k + 1}"] = xq[..., k].ravel()
            s = evaluate(model.source_plan(), b)
            if s.shape[1] != xq.shape[0] * xq.shape[1]:
                s = np.broadcast_to(s, (s.shape[0], xq.shape[0] * xq.shape[1]))
            if not np.isfinite(s).all():
                col = int(np.argwhere(~np.isfinite(s))[0][1])
                raise KernelNanError("source kernel produced non-finite values "
                                     f"(first at element {c0 + col // xq.shape[1]})")
            s = s.reshape(self.ncu, e.size, -1)                       # (c, e, q)
            wd = self.detj[e][:, None] * m.quad_wts[None, :]
            out[e] = -np.einsum("eq,ceq,qa->eac", wd, s, m.phi)
        return out


# ---------------------------------------------------------------------------
# dense (simplex) tables
# ---------------------------------------------------------------------------


def _face_vertex_perms(kind):
    import itertools
    nv = 2 if kind == "tri" else 3
    return [list(p) for p in itertools.permutations(range(nv))]


class DenseTables:
    """Host arrays for the dense-tabulation kernels (tri / tet): the
    reference's quadrature-point formulation (disc.py:436-821) with
    per-element affine geometry and orientation-indexed right traces
    instead of the reference's per-face Newton-inverted tabulations
    (disc.py:182-225; they agree to ~1e-15)."""

    def __init__(self, model, mesh, topo, master):
        self.model, self.mesh, self.topo, self.master = model, mesh, topo, master
        kind = master.kind
        if kind != mesh.elem_kind:
            raise DiscError("master element kind does not match the mesh")
        if kind not in ("tri", "tet"):
            raise DiscError(f"dense path is for simplices, got {kind}")
        if model.kind != "D":
            raise DiscError(f"B200 path supports diffusion (kind D) models, got {model.kind}")
        if model.nw > 0 or model.numflux.uhat is not None or model.numflux.fhat is not None:
            raise DiscError("ODE blocks and u^/f^ overrides are not supported on the B200 path")
        if master.quad_degree < 2 * master.p:
            raise DiscError("dense path needs quadrature degree >= 2p")
        self.kind = kind
        self.nd, self.p, self.ncu = mesh.nd, master.p, model.ncu
        self.nb = master.n_nodes
        self.nf = master.n_faces
        self.nqf = master.faces[0].weights.shape[0]
        self.ne = mesh.connectivity.shape[0]
        if self.ncu > 3:
            raise DiscError("dense path supports ncu <= 3")
        TensorTables._flux_coefficients(self)
        self._geometry()
        self._operators()
        self._faces()

    # reuse the affine geometry and face-geometry helpers of the tensor tables
    _geometry = TensorTables._geometry
    node_coords = TensorTables.node_coords
    face_normal_area = TensorTables.face_normal_area
    _switch_bits = TensorTables._switch_bits

    def _operators(self):
        m = self.master
        nd = self.nd
        dn = m.eval_basis_grad(m.nodes)                       # (a, b, r) = d phi_b / d xi_r (x_a)
        self.dr = np.ascontiguousarray(dn.transpose(2, 0, 1))  # (r, a, b)
        w = m.quad_wts
        self.kr = np.einsum("q,qar,qb->rab", w, m.dphi, m.phi)
        Mref = np.einsum("q,qa,qb->ab", w, m.phi, m.phi)
        self.minv = np.linalg.inv(Mref)
        self.lift = np.stack([self.minv @ (f.phi.T * f.weights[None, :]) for f in m.faces])
        self.fluxop = np.stack([f.phi.T * f.weights[None, :] for f in m.faces])
        self.phif = np.stack([f.phi for f in m.faces])       # own traces (nf, nqf, nb)
        # neighbour traces per (local face, vertex permutation of the face)
        perms = _face_vertex_perms(self.kind)
        self.perms = perms
        sigma = m.faces[0].sigma
        po = np.zeros((self.nf, len(perms), self.nqf, self.nb))
        self.perm_pts = np.zeros((self.nf, len(perms), self.nqf, nd))
        for lf in range(self.nf):
            v = refelem.VERTS[self.kind][list(refelem.FACES[self.kind][lf])]
            for o, pi in enumerate(perms):
                vp = v[pi]
                xi = vp[0][None, :] + sigma @ (vp[1:] - vp[0])
                self.perm_pts[lf, o] = xi
                po[lf, o] = m.eval_basis(xi)
        self.phio = po
        self.face_area_ref = np.array([m.faces[lf].weights.sum() for lf in range(self.nf)])

    def _faces(self):
        topo, model, mesh, m = self.topo, self.model, self.mesh, self.master
        ne, nf = self.ne, self.nf
        el, fl, er, fr = (np.asarray(a, dtype=np.int64) for a in
                          (topo.elem_l, topo.face_l, topo.elem_r, topo.face_r))
        nfi = el.size
        # per element-face outward normal and |t1 x t2| (read below for the
        # interior / boundary h and tau too)
        self.fnorm = np.zeros((ne, nf, self.nd))
        self.fsj = np.zeros((ne, nf))
        for lf in range(nf):
            n, sj = self.face_normal_area(np.arange(ne), lf)
            self.fnorm[:, lf] = n
            self.fsj[:, lf] = sj
        wsum = np.array([m.faces[lf].weights.sum() for lf in range(nf)])
        self.switch = self._switch_bits(el, fl)
        fnbr = np.full((ne, nf), -1, dtype=np.int32)
        finfo = np.full((ne, nf), -1, dtype=np.int32)
        ftau = np.zeros((ne, nf))
        tau = float(model.numflux.tau)
        over_h = True if model.numflux.tau_over_h is None else bool(model.numflux.tau_over_h)
        ws = model.wavespeed_plan()
        mu = model.mu_bindings()

        def lam(normals):
            # constant wavespeed folded into tau (linear path); the generated
            # path evaluates lambda(u) per face point on the device
            if ws is None or normals.shape[0] == 0 or self.nonlinear:
                return 0.0
            b = {"t": 0.0, **mu}
            for k in range(self.nd):
                b[f"n{k + 1}"] = normals[:, k]
            return evaluate(ws, b)[0]

        n_l = self.fnorm[el, fl]
        area = self.fsj[el, fl] * wsum[fl]
        fi_h = 0.5 * (self.elem_vol[el] + self.elem_vol[er]) / np.maximum(area, 1e-300)
        tau_i = (tau / fi_h if over_h else np.full(nfi, tau)) + lam(n_l)
        self.fi_h = fi_h
        # orientation: which vertex permutation of the neighbour's face lands
        # on this side's face quadrature points (periodic shift applied)
        tr = np.asarray(topo.translation, dtype=float)
        if tr.shape[0] != nfi:
            tr = np.zeros((nfi, self.nd))
        o_l = self._orient_fast(el, fl, er, fr, tr)
        o_r = self._orient_fast(er, fr, el, fl, -tr)
        sw = self.switch.astype(np.int32)
        fnbr[el, fl] = er
        fnbr[er, fr] = el
        finfo[el, fl] = (sw << 3) | (fr.astype(np.int32) << 4) | (o_l << 8)
        finfo[er, fr] = 4 | (sw << 3) | (fl.astype(np.int32) << 4) | (o_r << 8)
        ftau[el, fl] = tau_i
        ftau[er, fr] = tau_i
        eb, fb, tb = (np.asarray(a, dtype=np.int64) for a in
                      (topo.elem_b, topo.face_b, topo.tag_b))
        self.bc_groups = []
        for tag in (np.unique(tb) if tb.size else []):
            tag = int(tag)
            if tag not in model.bcs:
                raise DiscError(f"mesh boundary tag {tag} has no [bc] entry")
            bc = model.bcs[tag]
            if bc.type == "absorbing" and model.kind != "W":
                raise DiscError("absorbing boundaries require a wave model")   # disc.py:300-301
            if bc.type not in ("dirichlet", "neumann") and not (
                    self.nonlinear and bc.type == "absorbing"):
                raise DiscError(f"boundary type {bc.type!r} is not supported on the B200 path")
            self.bc_groups.append((tag, bc, np.nonzero(tb == tag)[0]))
        kinds = np.zeros(eb.size, dtype=np.int32)
        for tag, bc, idx in self.bc_groups:
            kinds[idx] = {"dirichlet": 1, "neumann": 2, "absorbing": 3}[bc.type]
        nb_ = self.fnorm[eb, fb]
        area_b = self.fsj[eb, fb] * wsum[fb]
        fb_h = self.elem_vol[eb] / np.maximum(area_b, 1e-300)
        if self.nd == 1:
            fb_h = self.elem_vol[eb]
        tau_b = (tau / fb_h if over_h else np.full(eb.size, tau)) + lam(nb_)
        self.fb_h = fb_h
        fnbr[eb, fb] = np.arange(eb.size, dtype=np.int32)
        finfo[eb, fb] = kinds
        ftau[eb, fb] = tau_b
        if np.any(finfo < 0):
            raise DiscError("element with an unclassified face")
        self.fnbr, self.finfo, self.ftau = fnbr, finfo, ftau
        self.n_boundary = eb.size
        self.eb, self.fb = eb, fb

    def face_points(self, elems, lf, pts=None):
        """Physical coordinates of face-lf quadrature points of elements."""
        xi = self.master.faces[lf].xi if pts is None else pts
        J = self.J[elems]                   # (e, d, r): one (e d) x r by r x q GEMM
        e, d = J.shape[0], J.shape[1]
        y = (J.reshape(e * d, -1) @ np.ascontiguousarray(xi.T)).reshape(e, d, -1)
        return self.x0[elems][:, None, :] + y.transpose(0, 2, 1)

    def _orient_fast(self, ea, fa, eb, fbb, shift):
        """_orient from the shared vertex ids where the two faces share
        their vertices (a conforming face: the permutation pi with
        ids_b[pi[i]] = ids_a[i] is the one whose points land on this side's,
        since both face maps are affine in the vertices); geometric matching
        only for the rest (periodic faces, whose vertices are translates)."""
        F = np.asarray(refelem.FACES[self.kind])
        conn = np.asarray(self.mesh.connectivity)
        nvf = F.shape[1]
        out = np.full(ea.size, -1, dtype=np.int32)
        if conn.shape[1] >= F.max() + 1 and ea.size:
            ga = conn[ea[:, None], F[fa]]
            gb = conn[eb[:, None], F[fbb]]
            eq = ga[:, :, None] == gb[:, None, :]
            ok = (eq.sum(axis=2) == 1).all(axis=1) & (eq.sum(axis=1) == 1).all(axis=1)
            pi = eq.argmax(axis=2)
            code = (pi * (nvf ** np.arange(nvf))).sum(axis=1)
            lut = np.full(nvf ** nvf, -1, dtype=np.int32)
            for o, p in enumerate(self.perms):
                lut[int(sum(v * nvf ** i for i, v in enumerate(p)))] = o
            out[ok] = lut[code[ok]]
        rest = np.nonzero(out < 0)[0]
        if rest.size:
            out[rest] = self._orient(ea[rest], fa[rest], eb[rest], fbb[rest], shift[rest])
        return out

    def _orient(self, ea, fa, eb, fbb, shift, chunk=1 << 15):
        n = ea.size
        out = np.full(n, -1, dtype=np.int32)
        scale2 = (1e-9 * max(self.mesh.diameter(), 1.0)) ** 2
        for a in range(self.nf):
            for b in range(self.nf):
                sel = np.nonzero((fa == a) & (fb_ == b))[0] if False else \
                    np.nonzero((fa == a) & (fbb == b))[0]
                for c0 in range(0, sel.size, chunk):
                    s = sel[c0:c0 + chunk]
                    x = self.face_points(ea[s], a) + shift[s][:, None, :]
                    for o in range(len(self.perms)):
                        todo = out[s] < 0
                        if not todo.any():
                            break
                        y = self.face_points(eb[s], b, self.perm_pts[b, o])
                        ok = np.sum((x - y) ** 2, axis=2).max(axis=1) <= scale2
                        out[s[ok & todo]] = o
        if np.any(out < 0):
            raise DiscError("could not orient a face (non-conforming mesh?)")
        return out

    def boundary_values(self, t):
        """(n_bfaces, nqf, ncu) Dirichlet / Neumann data at the face
        quadrature points (disc.py:559-563, 775-782)."""
        out = np.zeros((self.n_boundary, self.nqf, self.ncu))
        model = self.model
        for tag, bc, idx in self.bc_groups:
            if bc.type == "absorbing":
                continue
            plan = model.bc_plan(tag)
            for lf in range(self.nf):
                s = idx[self.fb[idx] == lf]
                if s.size == 0:
                    continue
                xq = self.face_points(self.eb[s], lf)
                n, _ = self.face_normal_area(self.eb[s], lf)
                b = {"t": float(t), **model.mu_bindings()}
                for k in range(self.nd):
                    b[f"x{k + 1}"] = xq[..., k].ravel()
                    b[f"n{k + 1}"] = np.repeat(n[:, k], xq.shape[1])
                g = evaluate(plan, b)
                if g.shape[1] != xq.shape[0] * xq.shape[1]:
                    g = np.broadcast_to(g, (g.shape[0], xq.shape[0] * xq.shape[1]))
                if not np.isfinite(g).all():
                    col = int(np.argwhere(~np.isfinite(g))[0][1])
                    raise KernelNanError(f"bc tag {tag} kernel produced non-finite values "
                                         f"(first at element {col // xq.shape[1]})")
                out[s] = g.reshape(self.ncu, s.size, -1).transpose(1, 2, 0)
        return out

    source_load = TensorTables.source_load
