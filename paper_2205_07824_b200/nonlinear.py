"""Generated-kernel LDG path for models the linear fused operator cannot take:
kind C (convection, local Lax-Friedrichs flux) and kind D models whose flux,
source, wavespeed or mass depend nonlinearly on the state (Euler,
compressible Navier-Stokes, Burgers, nonlinear diffusion...).

The model's plans are lowered to CUDA device functions (codegen.py), spliced
into ``csrc/ldg_nl.cuh`` with the element's compile-time shape and 1D
operators, and compiled once per (model, p, mesh kind) with NVRTC for sm_100a
(csrc/jit.cu).  Reference behaviour reproduced (ldgkit/disc.py):

* residual: volume flux and source by the element's Gauss rule (the same
  2p+1 rule as the reference), numerical fluxes at the face Gauss points
  (``_interior_fhat`` :657-699, ``_llf_flux`` :724-751, ``_boundary_fhat``
  :762-837, ``_llf_boundary`` :839-862), lifted with the face basis;
* tangent: the same code path on forward duals (expr.py:553-651), penalty
  frozen, LLF dlambda by the ``lam_l >= lam_r`` tie rule, boundary LLF
  dlambda only from the interior side, homogeneous lift, zero Neumann
  tangent (disc.py:591-604, :694-698, :745-751, :776-777, :806-818, :861);
* mixed gradient, mass, mass tangent extra and mass inverse
  (disc.py:436-490, :897-948; driver.py:92-106).

Scope: quad / hex, affine elements, conforming faces; Dirichlet and Neumann
boundaries (absorbing needs kind W, which raises, like ODE blocks and u^ / f^
overrides).  Face plans that read x on periodic meshes raise (the right
element would see the translated point).
"""

from __future__ import annotations

import ctypes as C
import hashlib
from pathlib import Path

import numpy as np

from . import _lib, codegen
from .expr import evaluate
from .tables import FACE_AXIS, DiscError, KernelNanError, TensorTables, affine_form, \
    plan_is_zero, uses_any

TEMPLATE = Path(__file__).resolve().parent / "csrc" / "ldg_nl.cuh"
# 3D element kernels: threads per element and faces per batch of the face
# phase.  Batches of 2 (opposite faces) need a third of the trace buffer, so
# 4-5 blocks fit an SM, but measured slower on the config-4 NS tangent (3.15 -
# 3.72 vs 4.23 GDOF/s, scripts/nl_ab.py, profiles/r2_nl_launch_shape_ab.jsonl):
# a batch's 32 face points leave 3 of 4 warps idle in the flux sweep
NT_3D = 128
FACE_BATCH_3D = 6
MINB_3D = 3                 # blocks per SM the 3D residual / tangent kernels are register-capped for
# 2D kind-C models (one warp per element): residual and uncached tangent
# capped to 24 blocks / SM (config-2 Euler p = 4, scripts/nl_ab.py: tangent
# 15.8 -> 17.0 GDOF/s, residual 25.0 -> 26.7; 32 blocks: 15.2 / 27.1;
# profiles/r2_nl_launch_shape_ab.jsonl); other 2D models keep the compiler's
# choice
MINB_2D_C = 24
LOAD_BATCH = 10             # element-load loads in flight per thread (NL_LOAD_BATCH; NS 3D tangent 4.23 -> 4.40 GDOF/s)


class NlParams(C.Structure):
    _fields_ = [("ne", C.c_int32), ("nbface", C.c_int32), ("t", C.c_double),
                ("scale", C.c_double)] + [(k, C.c_void_p) for k in (
                    "geo", "xmap", "fnbr", "finfo", "fgeo", "nmap", "gq", "gproj",
                    "u", "q", "du", "dq", "w", "dw", "out", "bad")] + [
                        ("homog", C.c_int32), ("pad_", C.c_int32)] + [(k, C.c_void_p) for k in (
                            "vgeo", "ffgeo", "minv", "bcache")]


def linear_path_reason(model):
    """None if the linear constant-coefficient fused path can run the model,
    else why the generated path is needed."""
    if model.kind != "D":
        return f"kind {model.kind}"
    if model.nw > 0:
        return "pointwise ODE block"
    if model.numflux.uhat is not None or model.numflux.fhat is not None:
        return "u^ / f^ override"
    if model.ncu > 3:
        return "ncu > 3"
    mu = model.mu_bindings()
    var = {f"u{i + 1}" for i in range(model.ncu)} | \
        {f"q{i + 1}_{j + 1}" for i in range(model.ncu) for j in range(model.nd)}
    forms = affine_form(model.flux_plan(), mu, var)
    if forms is None:
        return "flux not linear in (u, q) with constant coefficients"
    if any(abs(c) > 0 for _, c in forms):
        return "flux has a state-independent part"
    if uses_any(model.source_plan(), ("u", "q", "w")):
        return "state-dependent source"
    if affine_form(model.mass_plan(), mu, set()) is None:
        return "state-dependent mass"
    ws = model.wavespeed_plan()
    if ws is not None and uses_any(ws, ("u", "q", "w", "x")):
        return "state- or x-dependent wavespeed"
    return None


def _arr(a, name):
    return "{" + ", ".join(codegen.literal(v) for v in np.ravel(a)) + "}"


class NlTables(TensorTables):
    """TensorTables plus what the generated kernels read: the affine map
    x = x0 + J xi, per element-face (left normal, left |t1 x t2|, tau or
    tau/h), and the volume / face quadrature matched to the reference's
    rules (master.py quadrature, disc.py:139-180 face geometry)."""

    def __init__(self, model, mesh, topo, master):
        super().__init__(model, mesh, topo, master, nonlinear=True)
        m = self.master
        self.nq1 = len(m.quad1d[0])
        self._check_quadrature()
        nd, nf = self.nd, self.nf
        self.xmap = np.concatenate([self.x0, self.J.reshape(self.ne, -1)], axis=1)
        fgeo = np.zeros((self.ne, nf, nd + 2))
        t = self.topo
        el, fl, er, fr = (np.asarray(a, dtype=np.int64) for a in
                          (t.elem_l, t.face_l, t.elem_r, t.face_r))
        for e_, f_ in ((el, fl), (er, fr)):
            fgeo[e_, f_, :nd] = self.n_left
            fgeo[e_, f_, nd] = self.sj_left
            fgeo[e_, f_, nd + 1] = self.tau_i
        fgeo[self.eb, self.fb, :nd] = self.n_bnd
        fgeo[self.eb, self.fb, nd] = self.sj_bnd
        fgeo[self.eb, self.fb, nd + 1] = self.tau_b
        self.fgeo = fgeo
        tr = np.asarray(t.translation, dtype=float)
        self.periodic = tr.size > 0 and bool(np.any(tr != 0.0))
        if self.curved:
            self._curved_tables(el, fl, er, fr, tr)

    def _curved_tables(self, el, fl, er, fr, tr):
        """Per-point geometry of non-affine elements for the CURVED kernels:
          vgeo  (ne, NQ, 1 + nd^2 + nd): detJ, invJ^T, x at the volume points
          ffgeo (ne, nf, NQF, 2 nd + 1): per face point (kernel order) the
                LEFT element's unit normal, weight x |t1 x t2| and x at the
                physically matching left point -- both sides of an interior
                face evaluate f^ on bitwise identical inputs, as the
                reference's scatter of +/- one value (disc.py:641-653)
          minv  (ne, nb, nb): inverse element mass matrices (disc.py:107-110)."""
        m, nd, ne, nf = self.master, self.nd, self.ne, self.nf
        if self.model.kind not in ("C", "D") or self.model.nw > 0 or \
                self.model.numflux.uhat is not None:
            raise DiscError("curved elements are supported for kind C / D models without "
                            "ODE blocks or u^ overrides on the B200 path")
        self.vgeo = np.concatenate([self.detj_q[..., None], self.invjt_q.reshape(ne, -1, nd * nd),
                                    self.xq_q], axis=2)
        nqf = self.fxi.shape[1]
        ffgeo = np.zeros((ne, nf, nqf, 2 * nd + 1))

        def pack(x, n, mag, lf):
            return np.concatenate([n, (self.fw[lf][None, :] * mag)[..., None], x], axis=2)

        scale2 = (1e-9 * max(self.mesh.diameter(), 1.0)) ** 2
        for lf in range(nf):
            sel = np.nonzero(fl == lf)[0]
            if sel.size:
                x, n, mag = self.face_point_geometry(el[sel], lf, self.fxi[lf])
                ffgeo[el[sel], lf] = pack(x, n, mag, lf)
        for lf in range(nf):
            sel = np.nonzero(fr == lf)[0]
            if sel.size == 0:
                continue
            xr, _, _ = self.face_point_geometry(er[sel], lf, self.fxi[lf])
            left = ffgeo[el[sel], fl[sel]]                      # (k, nqf, 2nd+1)
            xl = left[..., nd + 1:] + (tr[sel][:, None, :] if tr.shape[0] == el.size else 0.0)
            d2 = ((xr[:, :, None, :] - xl[:, None, :, :]) ** 2).sum(axis=-1)
            j = d2.argmin(axis=2)
            if np.take_along_axis(d2, j[..., None], axis=2).max() > scale2:
                raise DiscError("curved face points do not match across an interior face")
            ffgeo[er[sel], lf] = np.take_along_axis(left, j[..., None], axis=1)
        for lf in range(nf):
            s_ = np.nonzero(self.fb == lf)[0]
            if s_.size:
                x, n, mag = self.face_point_geometry(self.eb[s_], lf, self.fxi[lf])
                ffgeo[self.eb[s_], lf] = pack(x, n, mag, lf)
        self.ffgeo = ffgeo
        self.minv = np.linalg.inv(np.einsum("eq,qa,qb->eab", self.wdetj_q, m.phi, m.phi))

    def _check_quadrature(self):
        """The reference's volume rule is the tensor Gauss rule (x fastest)
        and its face rules are tensor rules on the face; build the face-point
        tables in this kernel's ordering (tangential axes ascending) with the
        reference's own weights."""
        m, nd, nq1 = self.master, self.nd, self.nq1
        x1, w1 = m.quad1d
        idx = np.arange(nq1 ** nd)
        pts = np.stack([x1[(idx // nq1 ** k) % nq1] for k in range(nd)], axis=1)
        if m.quad_pts.shape != pts.shape or np.max(np.abs(m.quad_pts - pts)) > 1e-14:
            raise DiscError("generated path needs the tensor Gauss volume rule")
        wt = np.prod(np.stack([w1[(idx // nq1 ** k) % nq1] for k in range(nd)]), axis=0)
        if np.max(np.abs(m.quad_wts - wt)) > 1e-14:
            raise DiscError("volume weights are not the tensor Gauss weights")
        nqf = nq1 ** (nd - 1)
        fxi = np.zeros((self.nf, nqf, nd))
        fw = np.zeros((self.nf, nqf))
        for lf in range(self.nf):
            ax, hi = FACE_AXIS[m.kind][lf]
            tang = [a for a in range(nd) if a != ax]
            s = np.arange(nqf)
            my = np.zeros((nqf, nd))
            my[:, ax] = 1.0 if hi else -1.0
            for k, a in enumerate(tang):
                my[:, a] = x1[(s // nq1 ** k) % nq1]
            ref = m.faces[lf].xi
            d = np.abs(my[:, None, :] - ref[None, :, :]).max(axis=2)
            j = np.argmin(d, axis=1)
            if d[s, j].max() > 1e-13 or np.unique(j).size != nqf or ref.shape[0] != nqf:
                raise DiscError("face quadrature is not the tensor Gauss rule")
            fxi[lf] = ref[j]
            fw[lf] = m.faces[lf].weights[j]
        self.fxi, self.fw = fxi, fw

    # -- time-dependent boundary data at the face Gauss points (own frame) --
    def boundary_points(self, t):
        """(n_bfaces, nqf, ncu) values of each Dirichlet / Neumann plan at
        the boundary face's Gauss points (disc.py:762-837 evaluate the bc
        plans at fb_x with the boundary normal)."""
        nbf = self.n_boundary
        nqf = self.fxi.shape[1]
        out = np.zeros((nbf, nqf, self.ncu))
        mu = self.model.mu_bindings()
        for tag, bc, idx in self.bc_groups:
            if bc.type == "absorbing":
                continue
            plan = self.model.bc_plan(tag)
            for lf in range(self.nf):
                s = idx[self.fb[idx] == lf]
                if s.size == 0:
                    continue
                e = self.eb[s]
                if self.curved:
                    ff = self.ffgeo[e, lf]
                    xq, nq = ff[..., self.nd + 1:], ff[..., :self.nd]
                else:
                    xq = self.x0[e][:, None, :] + np.einsum("edr,qr->eqd", self.J[e],
                                                            self.fxi[lf])
                    nq = np.repeat(self.n_bnd[s][:, None, :], nqf, axis=1)
                b = {"t": float(t), **mu}
                for k in range(self.nd):
                    b[f"x{k + 1}"] = xq[..., k].ravel()
                    b[f"n{k + 1}"] = nq[..., k].ravel()
                g = evaluate(plan, b)
                if g.shape[1] != s.size * nqf:
                    g = np.broadcast_to(g, (g.shape[0], s.size * nqf))
                if not np.isfinite(g).all():
                    col = int(np.argwhere(~np.isfinite(g))[0][1])
                    raise KernelNanError(f"bc tag {tag} kernel produced non-finite "
                                         f"values (first at element {col // nqf})")
                out[s] = g.reshape(self.ncu, s.size, nqf).transpose(1, 2, 0)
        return out


def generate_source(tab):
    """Full NVRTC source of the model's kernels (prelude + plans + template)."""
    model, m = tab.model, tab.master
    nd, ncu = tab.nd, tab.ncu
    mu = model.mu_bindings()
    flux, src = model.flux_plan(), model.source_plan()
    ws, mass = model.wavespeed_plan(), model.mass_plan()
    if codegen.uses(flux, "n"):
        raise DiscError("flux plans may not read the normal (the reference binds none "
                        "at volume points)")
    if model.kind == "C" and codegen.uses(flux, "q"):
        raise DiscError("kind C fluxes cannot read q")
    if model.kind == "C" and ws is None:
        raise DiscError("kind C models need a wavespeed for the LLF flux")
    if ws is not None and (codegen.uses(ws, "q") or codegen.uses(ws, "w")):
        raise DiscError("wavespeed plans may read x, t, u, n only")
    if codegen.uses(mass, "q") or codegen.uses(mass, "w"):
        raise DiscError("the mass may read x, t, u only on the generated path")
    absorbing = any(bc.type == "absorbing" for _, bc, _ in tab.bc_groups)
    if absorbing and (ws is None or codegen.uses(ws, "u") or codegen.uses(ws, "x")):
        raise DiscError("absorbing boundaries need a wavespeed independent of u and x "
                        "(the gradient lift takes u^ at the face nodes)")
    nw = model.nw
    sw = model.sw_plan() if nw > 0 else None
    uhat, fhat = model.uhat_plan(), model.fhat_plan()
    if tab.periodic and any(p is not None and codegen.uses(p, "x") for p in (uhat, fhat)):
        raise DiscError("face override plans reading x on periodic meshes are not supported")
    if uhat is not None:
        # the gradient lift takes u^ at the face nodes: exact for u^ affine in
        # the traces with constant coefficients (no q, no x)
        face_vars = {f"u{s}{i + 1}" for s in "lr" for i in range(ncu)}
        if affine_form(uhat, mu, face_vars) is None:
            raise DiscError("u^ overrides must be affine in ul / ur with constant coefficients")
    if tab.periodic and (codegen.uses(flux, "x") or (ws is not None and codegen.uses(ws, "x"))):
        raise DiscError("face plans reading x on periodic meshes are not supported")
    mforms = affine_form(mass, mu, set())
    mass_const = mforms is not None
    n1, nq1 = tab.n1, tab.nq1
    nvq = 0 if model.kind == "C" else ncu * nd
    nv = ncu + nvq + nw
    kmax = max(n1, nq1)
    mx, mxf = kmax ** nd, kmax ** (nd - 1)
    nq, nb = nq1 ** nd, n1 ** nd
    # threads per element: the quadrature points rounded to warps; 3D elements
    # get at least 128 (contractions and face work have more parallelism)
    nt = min(256, ((max(nq, nb) + 31) // 32) * 32)
    if nd == 3:
        nt = max(nt, NT_3D)
    fb = FACE_BATCH_3D if nd == 3 else 2 * nd
    kind_c2 = nd == 2 and model.kind == "C"
    ng = ncu * (nd + 1)
    ode = model.ode
    defs = dict(ND=nd, N1=n1, NQ1=nq1, NCU=ncu, NW=nw, KIND_C=int(model.kind == "C"),
                KIND_W=int(model.kind == "W"),
                ODE_ALPHA=codegen.literal(ode.alpha if ode is not None else 1.0),
                ODE_BETA=codegen.literal(ode.beta if ode is not None else 0.0),
                HAS_WS=int(ws is not None), TRACE_CENTERED=int(model.numflux.trace == "centered"),
                GRAD_CENTERED=int(model.numflux.grad_trace == "centered"),
                HAS_UHAT=int(uhat is not None), HAS_FHAT=int(fhat is not None),
                MASS_CONST=int(mass_const), NT=nt, CURVED=int(bool(getattr(tab, "curved", False))),
                NL_FB=fb, NL_RES_MINB=MINB_3D if nd == 3 else (MINB_2D_C if kind_c2 else 1),
                NL_TAN_MINB=MINB_3D if nd == 3 else 1, NL_LOAD_BATCH=LOAD_BATCH)
    if kind_c2:
        defs["NL_TANU_MINB"] = MINB_2D_C
    lines = ["// generated by paper_2205_07824_b200/nonlinear.py -- do not edit"]
    lines += [f"#define {k} {v}" for k, v in defs.items()]
    mc = np.zeros(ncu)
    if mass_const:
        mc[:] = [f[1] for f in mforms]
    consts = dict(c_phi=m.phi1d, c_dphi=m.dphi1d, c_d1=tab.d1, c_clo=tab.clo, c_chi=tab.chi,
                  c_m1inv=tab.m1inv, c_xq1=m.quad1d[0], c_qw=m.quad_wts, c_fxi=tab.fxi,
                  c_fw=tab.fw, c_mass=mc, c_xn=m.nodes)
    for k, v in consts.items():
        lines.append(f"__constant__ double {k}[{np.size(v)}] = {_arr(v, k)};")
    lines.append(codegen.DEVICE_HELPERS)
    lines.append(codegen.emit_plan(flux, "plan_flux", nd, mu))
    lines.append(codegen.emit_plan(src, "plan_src", nd, mu))
    if ws is not None:
        lines.append(codegen.emit_plan(ws, "plan_ws", nd, mu))
    else:
        lines.append(codegen.emit_plan(_ZeroPlan(1), "plan_ws", nd, mu))
    lines.append(codegen.emit_plan(mass, "plan_mass", nd, mu))
    lines.append(codegen.emit_plan(sw if sw is not None else _ZeroPlan(1), "plan_sw", nd, mu))
    lines.append(codegen.emit_face_plan(uhat if uhat is not None else _ZeroPlan(ncu),
                                        "plan_uhat", nd, mu))
    lines.append(codegen.emit_face_plan(fhat if fhat is not None else _ZeroPlan(ncu),
                                        "plan_fhat", nd, mu))
    src_text = "\n".join(lines) + "\n" + TEMPLATE.read_text()
    shapes = dict(defs, NB=nb, NQ=nq, NV=nv, MX=mx, MXF=mxf, NG=ng)
    return src_text, shapes


class _ZeroPlan:
    def __init__(self, n):
        self.instructions = (("const", 0.0),)
        self.outputs = (0,) * n


_CUBINS = {}


def compile_source(src):
    """NVRTC -> CUBIN bytes (cached per source text)."""
    key = hashlib.sha256(src.encode()).hexdigest()
    if key in _CUBINS:
        return _CUBINS[key]
    lib = _lib.load(require_gpu=False)
    size = C.c_int64(0)
    b = src.encode()
    _lib.check(lib.ldg_jit_compile(b, b"ldg_nl.cu", None, 0, None, C.byref(size)),
               "ldg_jit_compile", jit=True)
    buf = C.create_string_buffer(size.value)
    _lib.check(lib.ldg_jit_compile(b, b"ldg_nl.cu", None, 0, buf, C.byref(size)),
               "ldg_jit_compile", jit=True)
    _CUBINS[key] = buf.raw[: size.value]
    return _CUBINS[key]


class NlOperator:
    """Device tables + the loaded module of one system's generated kernels."""

    def __init__(self, tab, device):
        import torch
        self.tab, self.device = tab, device
        self.src, self.shape = generate_source(tab)
        self.cubin = compile_source(self.src)
        self.lib = _lib.load()
        h = C.c_void_p()
        _lib.check(self.lib.ldg_jit_load(self.cubin, len(self.cubin), C.byref(h)),
                   "ldg_jit_load", jit=True)
        self._mod = h

        def dev(a, dt):
            return torch.as_tensor(np.ascontiguousarray(a, dtype=dt), device=device)

        self.geo = dev(tab.geo, np.float64)
        self.xmap = dev(tab.xmap, np.float64)
        self.fnbr = dev(tab.fnbr, np.int32)
        self.finfo = dev(tab.finfo, np.int32)
        self.fgeo = dev(tab.fgeo, np.float64)
        self.nmap = dev(tab.nmap, np.int32)
        curved = getattr(tab, "curved", False)
        self.vgeo = dev(tab.vgeo, np.float64) if curved else None
        self.ffgeo = dev(tab.ffgeo, np.float64) if curved else None
        self.minv = dev(tab.minv, np.float64) if curved else None
        self.bad = torch.full((1,), -1, dtype=torch.int64, device=device)
        self._bq, self._bp = {}, {}
        s = self.shape
        nv, nb, mx, ng, ncu = s["NV"], s["NB"], s["MX"], s["NG"], tab.ncu
        self.smem = {}
        nd, nqf, mxf = tab.nd, tab.nq1 ** (tab.nd - 1), s["MXF"]
        for name, nva in (("nl_residual", nv), ("nl_tangent", 2 * nv), ("nl_tangent_cached", nv),
                          ("nl_base_cache", nv)):
            nbf = nva * s["NB"] // s["N1"]          # one face's neighbour nodes (NVA x NFN)
            fb = s["NL_FB"]                         # faces per batch of the face phase
            face = 2 * fb * nva * nqf + nbf + 2 * nva * mxf + fb * nqf * ncu + 2 * nbf
            work = max(2 * max(nva, ng) * mx + 2 * nbf, face)
            self.smem[name] = 8 * (nva * nb + ncu * nb + work)
        nvm = ncu if s["MASS_CONST"] else 3 * ncu
        self.smem["nl_mass"] = self.smem["nl_mass_extra"] = 8 * 2 * max(nvm, ncu) * mx
        self.smem["nl_mass_inv"] = 8 * 2 * ncu * nb
        ngq, nqf_ = ncu * nd, tab.nq1 ** (nd - 1)
        mcs = max(ngq, ncu) * mx
        self.smem["nl_mixed_curved"] = 8 * (ncu * nb + 3 * mcs + ngq * nb + 2 * 2 * nd * ncu * nqf_
                                            + 4 * ncu * mxf + 2 * nd * nqf_ * ngq)
        self.smem["nl_mass_q"] = 8 * 2 * ncu * tab.nd * mx
        self.smem["nl_mass_inv_q"] = 8 * 2 * ncu * tab.nd * nb

    def __del__(self):
        h = getattr(self, "_mod", None)
        if h is not None and getattr(self, "lib", None) is not None:
            try:
                self.lib.ldg_jit_unload(h)
            except Exception:
                pass

    # -- boundary data (cached per t) -----------------------------------------
    def gq(self, t):
        import torch
        key = float(t)
        if key not in self._bq:
            if len(self._bq) > 4:
                self._bq.clear()
            g = self.tab.boundary_points(key)
            self._bq[key] = torch.as_tensor(g, device=self.device) if g.size else None
        return self._bq[key]

    def gproj(self, t):
        import torch
        key = float(t)
        if key not in self._bp:
            if len(self._bp) > 4:
                self._bp.clear()
            g = self.tab.boundary_projection(key)
            self._bp[key] = torch.as_tensor(g, device=self.device) if g.size else None
        return self._bp[key]

    def _launch(self, name, grid, block, P):
        smem = self.smem.get(name, 0)
        _lib.check(self.lib.ldg_jit_launch(self._mod, name.encode(), grid, 1, block, smem,
                                           C.byref(P), C.sizeof(P), _lib.stream_ptr()),
                   name, jit=True)

    def _params(self, t=0.0, scale=1.0, **ptrs):
        P = NlParams()
        P.ne, P.nbface, P.t, P.scale = self.tab.ne, self.tab.n_boundary, float(t), float(scale)
        for k in ("geo", "xmap", "fnbr", "finfo", "fgeo", "nmap"):
            setattr(P, k, getattr(self, k).data_ptr())
        for k in ("vgeo", "ffgeo", "minv"):
            v = getattr(self, k)
            setattr(P, k, None if v is None else v.data_ptr())
        P.bad = self.bad.data_ptr()
        for k, v in ptrs.items():
            setattr(P, k, None if v is None else v.data_ptr())
        return P

    def _empty(self, shape):
        import torch
        return torch.empty(shape, dtype=torch.float64, device=self.device)

    # -- operators -------------------------------------------------------------
    def mixed(self, u, t=0.0, homogeneous=False, out=None, state_q=None, linearised=False):
        """M^-1 (lifted gradient form) of u; `state_q` (kind W) is the state
        gradient absorbing boundaries take u^ from."""
        tab = self.tab
        q = out if out is not None else self._empty((tab.ne, self.shape["NB"], tab.ncu, tab.nd))
        if getattr(tab, "curved", False):
            # quadrature form with per-point metrics and M_e^-1 (disc.py:436-490)
            P = self._params(t, u=u, out=q, gq=None if homogeneous else self.gq(t))
            self._launch("nl_mixed_curved", tab.ne, self.shape["NT"], P)
            return q
        P = self._params(t, u=u, q=state_q, out=q,
                         gproj=None if homogeneous else self.gproj(t))
        P.homog = int(bool(linearised))
        nb = self.shape["NB"]
        epb = 1 if nb >= 128 else 128 // nb
        self._launch("nl_mixed", (tab.ne + epb - 1) // epb, epb * nb, P)
        return q

    def residual(self, u, t=0.0, q=None, w=None, out=None):
        """Ru; q is the state gradient (kind W) or the mixed gradient (kind D,
        computed when not given); w the ODE states."""
        R = out if out is not None else self._empty(u.shape)
        if self.tab.model.kind == "D" and q is None:
            q = self.mixed(u, t)
        P = self._params(t, u=u, q=q, w=w, out=R, gq=self.gq(t))
        self._launch("nl_residual", self.tab.ne, self.shape["NT"], P)
        return R

    def base_cache(self, u, t=0.0, q=None, w=None):
        """The tangent's loop-invariant half for one base state: u, q, w at
        the volume and face points (own and neighbour side), built once per
        base (a Newton step's GMRES matvecs and block-Jacobi probes share it)
        -- the base mixed gradient is cached the same way.  Keyed by the base
        tensors' identity and version and t."""
        import torch

        def tag(a):
            return None if a is None else (a.data_ptr(), a._version, tuple(a.shape))
        key = (tag(u), tag(q), tag(w), float(t))
        if getattr(self, "_bkey", None) == key:
            return self._bcache
        s = self.shape
        n = self.tab.ne * (s["NV"] * s["NQ"] + 2 * 2 * self.tab.nd * s["NV"] * self.tab.nq1 **
                           (self.tab.nd - 1))
        if getattr(self, "_bcache", None) is None or self._bcache.numel() != n:
            self._bcache = torch.empty(n, dtype=torch.float64, device=self.device)
        P = self._params(t, u=u, q=q, w=w, bcache=self._bcache)
        self._launch("nl_base_cache", self.tab.ne, s["NT"], P)
        # the entry holds the base tensors themselves, so their storage cannot
        # be recycled by the allocator for another state at the same address
        self._bkey, self._bkeep = key, (u, q, w)
        return self._bcache

    def tangent(self, u, du, t=0.0, q=None, w=None, dq=None, dw=None, out=None, cached=None):
        """dRu (the reference linearisation); kind D derives dq from du by
        the homogeneous lift, kind W takes the state direction dq.  With
        `cached` the base state's point values come from base_cache() and
        only the direction is interpolated."""
        R = out if out is not None else self._empty(du.shape)
        if self.tab.model.kind == "D":
            if q is None:
                q = self.mixed(u, t)
            if dq is None:                         # (partitioned callers pass it with halos)
                dq = self.mixed(du, t, homogeneous=True)
        if cached is None:
            # measured: 3D kind D (Navier-Stokes: 20 base variables) 2.58 ->
            # 3.69 GDOF/s; 2D Euler (4) 15.7 -> 14.2 -- the cache pays where
            # the base interpolation is large
            cached = self.tab.model.kind == "D" and self.tab.nd == 3
        if cached:
            bc = self.base_cache(u, t, q, w)
            P = self._params(t, u=u, q=q, du=du, dq=dq, w=w, dw=dw, out=R, gq=self.gq(t),
                             bcache=bc)
            self._launch("nl_tangent_cached", self.tab.ne, self.shape["NT"], P)
            return R
        P = self._params(t, u=u, q=q, du=du, dq=dq, w=w, dw=dw, out=R, gq=self.gq(t))
        self._launch("nl_tangent", self.tab.ne, self.shape["NT"], P)
        return R

    def gradient_residual(self, u, q, t=0.0, tangent=False, out=None):
        """Kind W gradient equation, Rq = -(lifted gradient form)
        (disc.py:866-874): the lift of (u, q) -- or of the direction (du, dq)
        with homogeneous Dirichlet data -- times the element mass."""
        tab = self.tab
        qt = self.mixed(u, t, homogeneous=tangent, state_q=q, linearised=tangent)
        o = out if out is not None else self._empty(qt.shape)
        P = self._params(t, -1.0, q=qt, out=o)
        self._launch("nl_mass_q", tab.ne, self.shape["NT"], P)
        return o

    def mass_q(self, v, scale=1.0, out=None):
        o = out if out is not None else self._empty(v.shape)
        P = self._params(0.0, scale, q=v, out=o)
        self._launch("nl_mass_q", self.tab.ne, self.shape["NT"], P)
        return o

    def mass_inv_q(self, v, out=None):
        o = out if out is not None else self._empty(v.shape)
        P = self._params(0.0, 1.0, q=v, out=o)
        self._launch("nl_mass_inv_q", self.tab.ne, self.shape["NT"], P)
        return o

    def ode(self, u, q, w, t=0.0, du=None, dq=None, dw=None, out=None):
        """Rw = beta w - s_w (or its tangent when du is given), at the nodes."""
        tab = self.tab
        o = out if out is not None else self._empty(w.shape)
        P = self._params(t, u=u, q=q, w=w, du=du, dq=dq, dw=dw, out=o)
        n = tab.ne * self.shape["NB"]
        self._launch("nl_ode_tangent" if du is not None else "nl_ode", (n + 127) // 128, 128, P)
        return o

    def mass(self, v, u=None, t=0.0, scale=1.0, out=None):
        o = out if out is not None else self._empty(v.shape)
        if not self.shape["MASS_CONST"] and u is None:
            raise DiscError("state-dependent mass needs the base state")
        P = self._params(t, scale, q=v, u=u, out=o)
        self._launch("nl_mass", self.tab.ne, self.shape["NT"], P)
        return o

    def mass_extra(self, y, u, du, t=0.0, scale=1.0, out=None):
        o = out if out is not None else self._empty(y.shape)
        P = self._params(t, scale, q=y, u=u, du=du, out=o)
        self._launch("nl_mass_extra", self.tab.ne, self.shape["NT"], P)
        return o

    def mass_inv(self, v, scale=1.0, out=None):
        o = out if out is not None else self._empty(v.shape)
        P = self._params(0.0, scale, q=v, out=o)
        self._launch("nl_mass_inv", self.tab.ne, self.shape["NT"], P)
        return o

    def reset_bad(self):
        self.bad.fill_(-1)

    def bad_element(self):
        v = int(self.bad.item())
        return -1 if v == -1 else v

    def kernel_attrs(self, name):
        r, l, s = C.c_int(), C.c_int(), C.c_int()
        _lib.check(self.lib.ldg_jit_attr(self._mod, name.encode(), C.byref(r), C.byref(l),
                                         C.byref(s)), "ldg_jit_attr", jit=True)
        return {"regs": r.value, "local_bytes": l.value, "static_smem": s.value}
