"""Drop-in ``LdgSystem`` whose residual / tangent / mixed-gradient / mass
operators run as hand-written sm_100a CUDA kernels.

Mirrors ``ldgkit.disc.LdgSystem`` (disc.py:257-948): same constructor
(model, mesh, topology, master), same methods and return conventions
(tuples of block arrays; a new array per call), same error types and
messages (``DiscError``, ``KernelNanError("<label> kernel produced
non-finite values (first at element N)")``).  numpy inputs give numpy
outputs (host<->device copies included); torch CUDA tensors stay on the
device, which is how the device solver (``solver.py``) drives it.

There is no CPU path: constructing a system without the native library or
without a GPU raises.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .tables import DenseTables, DiscError, KernelNanError, TensorTables, mesh_is_affine
from .nonlinear import NlOperator, NlTables, linear_path_reason

# elements from which the volume source load is evaluated on the device (the
# host restatement costs ~15 us per element: 2.3 s at config 3's 157K hexes)
DEVICE_SOURCE_MIN_NE = 32768

__all__ = ["LdgSystem", "SolverState", "DiscError", "KernelNanError"]


@dataclass
class SolverState:
    """disc.py:45-66."""

    u: object
    q: object
    w: object
    t: float

    def copy(self):
        c = (lambda a: None if a is None else a.clone() if hasattr(a, "clone") else a.copy())
        return SolverState(c(self.u), c(self.q), c(self.w), self.t)

    def all_finite(self):
        import torch
        ok = True
        for a in (self.u, self.q, self.w):
            if a is None:
                continue
            ok = ok and bool(torch.isfinite(a).all()) if hasattr(a, "is_cuda") \
                else ok and bool(np.isfinite(a).all())
        return ok


class _Disc:
    """Host-side geometry views read by reference callers
    (driver.py:102, diagnostics.py:43-63): computed lazily from the affine
    tables, never used by the kernels."""

    def __init__(self, tab):
        self._t = tab

    @property
    def node_x(self):
        return self._t.node_coords()

    @property
    def wdetj(self):
        if getattr(self._t, "curved", False):
            return self._t.wdetj_q
        return self._t.detj[:, None] * self._t.master.quad_wts[None, :]

    @property
    def xq(self):
        t = self._t
        if getattr(t, "curved", False):
            return t.xq_q
        return t.x0[:, None, :] + np.einsum("edr,qr->eqd", t.J, t.master.quad_pts)

    @property
    def detj(self):
        if getattr(self._t, "curved", False):
            return self._t.detj_q
        return np.repeat(self._t.detj[:, None], self._t.master.quad_pts.shape[0], axis=1)

    @property
    def mass_inv(self):
        t = self._t
        if getattr(t, "curved", False):
            return t.minv
        if hasattr(t, "minv"):                      # simplex: M_e = detJ M_ref
            return t.minv[None, :, :] / t.detj[:, None, None]
        mi = t.m1inv
        k = np.kron(np.kron(mi, mi), mi) if t.nd == 3 else np.kron(mi, mi)
        return k[None, :, :] / t.detj[:, None, None]

    @property
    def fi_h(self):
        return self._t.fi_h

    @property
    def fb_h(self):
        return self._t.fb_h


class LdgSystem:
    """The semi-discrete LDG operator on the B200.

    Three device paths behind one interface: the fused sum-factorised
    operator (quad/hex, kind D, flux linear in (u, q) with constant
    coefficients: ldg_fused.cu), the dense simplex kernels (tri/tet,
    ldg_dense.cu) and the generated model-specific kernels (quad/hex, kind C
    or any nonlinear kind-D model: nonlinear.py + ldg_nl.cuh via NVRTC)."""

    def __init__(self, model, mesh, topology, master, device=None, tables=None):
        """`tables` (internal): prebuilt host tables, e.g. one partition's
        ``parallel.LocalTables``; default builds them from the setup objects."""
        import torch
        self.model, self.mesh, self.topology, self.master = model, mesh, topology, master
        self.kind = model.kind
        self.ncu, self.nd, self.nw = model.ncu, model.nd, model.nw
        if model.nd != mesh.nd:
            raise DiscError(f"model nd={model.nd} but mesh nd={mesh.nd}")
        self.dense = master.kind in ("tri", "tet")
        self.nl = None
        self.nl_reason = None if self.dense else linear_path_reason(model)
        if self.nl_reason is None and not self.dense and tables is None and \
                not mesh_is_affine(mesh):
            self.nl_reason = "curved (non-affine) elements"
        if self.nl_reason is None and mesh.nd == 1:
            self.nl_reason = "1D elements (the fused kernels are quad / hex)"
        if tables is not None and self.nl_reason is not None:
            raise DiscError(f"prebuilt (partitioned) tables support linear models only "
                            f"({self.nl_reason})")
        if tables is not None:
            self.tab = tables
        elif self.dense:
            self.tab = DenseTables(model, mesh, topology, master)
        elif self.nl_reason is not None:
            self.tab = NlTables(model, mesh, topology, master)
        else:
            self.tab = TensorTables(model, mesh, topology, master)
        self.lib = _lib.load()
        self.device = torch.device(device if device is not None else "cuda")
        self.fi_switch = self.tab.switch
        self.beta_hat = np.ones(mesh.nd) / np.sqrt(mesh.nd)
        self.bc_groups = self.tab.bc_groups
        self.disc = _Disc(self.tab)
        if self.nl_reason is not None:
            self.nl = NlOperator(self.tab, self.device)
            self._h = None
            self._baseq = None
        else:
            self._create_handle()
        self._bdata = {}
        self._src = {}
        self._devsrc = None
        if (not self.dense and self.nl is None and not getattr(self.tab, "source_zero", False)
                and getattr(self.tab, "x0", None) is not None and self.tab.ne >= DEVICE_SOURCE_MIN_NE
                and not getattr(self.tab, "curved", False)):
            # NVRTC-compile the source plan now (setup) rather than inside the
            # first residual of a solve
            from .source_dev import DeviceSource
            self._devsrc = DeviceSource(self.tab, self.device)
        self._scratch = {}

    # -- native handle -------------------------------------------------------------
    def _create_dense_handle(self):
        t = self.tab
        T = _lib.LdgDenseTables()
        T.nd, T.nb, T.nqf, T.nface = t.nd, t.nb, t.nqf, t.nf
        T.nperm, T.ncu, T.ne = len(t.perms), t.ncu, t.ne
        T.trace_centered = int(self.model.numflux.trace == "centered")
        T.grad_centered = int(self.model.numflux.grad_trace == "centered")
        T.flux_uses_u = int(t.flux_uses_u)
        keep = []

        def arr(a, dt):
            a, p = _lib.as_c(a, dt)
            keep.append(a)
            return p

        T.geo = arr(t.geo, np.float64)
        T.fnorm = arr(t.fnorm, np.float64)
        T.fsj = arr(t.fsj, np.float64)
        T.fnbr = arr(t.fnbr, np.int32)
        T.finfo = arr(t.finfo, np.int32)
        T.ftau = arr(t.ftau, np.float64)
        T.dr = arr(t.dr, np.float64)
        T.kr = arr(t.kr, np.float64)
        T.lift = arr(t.lift, np.float64)
        T.fluxop = arr(t.fluxop, np.float64)
        T.phif = arr(t.phif, np.float64)
        T.phio = arr(t.phio, np.float64)
        for k, v in enumerate(t.au.ravel()):
            T.au[k] = v
        for k, v in enumerate(t.aq.ravel()):
            T.aq[k] = v
        h = C.c_void_p()
        _lib.check(self.lib.ldg_create_dense(C.byref(T), C.byref(h)), "ldg_create_dense")
        self._h = h

    def _create_handle(self):
        if self.dense:
            return self._create_dense_handle()
        t = self.tab
        T = _lib.LdgTables()
        T.nd, T.n1, T.ncu, T.ne = t.nd, t.n1, t.ncu, t.ne
        T.n_maps = t.nmap.shape[0]
        T.trace_centered = int(self.model.numflux.trace == "centered")
        T.grad_centered = int(self.model.numflux.grad_trace == "centered")
        T.flux_uses_u = int(t.flux_uses_u)
        self._keep = []

        def arr(a, dt):
            a, p = _lib.as_c(a, dt)
            self._keep.append(a)
            return p

        T.geo = arr(t.geo, np.float64)
        T.fnbr = arr(t.fnbr, np.int32)
        T.finfo = arr(t.finfo, np.int32)
        T.ftau = arr(t.ftau, np.float64)
        T.nmap = arr(t.nmap, np.int32)
        n1 = t.n1
        for name in ("d1", "m1", "s1"):
            dst = getattr(T, name)
            src = np.ascontiguousarray(getattr(t, name)).ravel()
            for k in range(n1 * n1):
                dst[k] = src[k]
        for k in range(n1):
            T.clo[k] = t.clo[k]
            T.chi[k] = t.chi[k]
        for k, v in enumerate(t.au.ravel()):
            T.au[k] = v
        for k, v in enumerate(t.aq.ravel()):
            T.aq[k] = v
        for k, v in enumerate(t.mass_coef):
            T.mass_coef[k] = v
        h = C.c_void_p()
        _lib.check(self.lib.ldg_create(C.byref(T), C.byref(h)), "ldg_create")
        self._keep = None
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and getattr(self, "lib", None) is not None:
            try:
                self.lib.ldg_destroy(h)
            except Exception:
                pass

    # -- shapes and packing (disc.py:310-355) ----------------------------------------
    @property
    def n_elements(self):
        return self.tab.ne

    @property
    def n_nodes(self):
        return self.master.n_nodes

    def block_shapes(self):
        """disc.py:320-326: u, then q for kind W, then w for ODE blocks."""
        ne, nb = self.n_elements, self.n_nodes
        shapes = [("u", (ne, nb, self.ncu))]
        if self.kind == "W":
            shapes.append(("q", (ne, nb, self.ncu, self.nd)))
        if self.nw > 0:
            shapes.append(("w", (ne, nb, self.nw)))
        return shapes

    @property
    def multi_block(self):
        """True when the packed state carries q (kind W) or w (ODE) blocks."""
        return self.kind == "W" or self.nw > 0

    @property
    def n_dofs(self):
        return sum(int(np.prod(s)) for _, s in self.block_shapes())

    def pack(self, u, q=None, w=None):
        """disc.py:333-339 (numpy or torch)."""
        parts = [u]
        if self.kind == "W":
            parts.append(q)
        if self.nw > 0:
            parts.append(w)
        if hasattr(u, "is_cuda"):
            import torch
            if len(parts) == 1:
                return u.reshape(-1)
            return torch.cat([p.reshape(-1) for p in parts])
        return np.concatenate([np.ravel(p) for p in parts])

    def unpack(self, vec):
        """disc.py:341-351: views of the packed blocks."""
        out, k = [], 0
        for _, shape in self.block_shapes():
            n = int(np.prod(shape))
            out.append(vec[k:k + n].reshape(shape))
            k += n
        u = out[0]
        q = out[1] if self.kind == "W" else None
        w = out[-1] if self.nw > 0 else None
        return u, q, w

    def state_from_vector(self, vec, t):
        u, q, w = self.unpack(vec)
        return SolverState(u=u, q=q, w=w, t=t)

    # -- device helpers ----------------------------------------------------------------
    def _dev(self, a):
        """-> (device tensor, origin) with origin 'cuda', 'torch' (host
        torch tensor, returned as host torch) or 'numpy'."""
        import torch
        if isinstance(a, torch.Tensor):
            if a.is_cuda:
                return a.to(self.device, torch.float64).contiguous(), "cuda"
            pinned = a.is_pinned()
            return a.to(self.device, torch.float64, non_blocking=pinned).contiguous(), "torch"
        return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64),
                               device=self.device), "numpy"

    def _empty(self, shape):
        import torch
        return torch.empty(shape, dtype=torch.float64, device=self.device)

    def boundary_data(self, t):
        """Projected Dirichlet/Neumann data at time t (device, cached)."""
        import torch
        key = float(t)
        if key not in self._bdata:
            if len(self._bdata) > 4:
                self._bdata.clear()
            g = self.tab.boundary_values(key) if self.dense else \
                self.tab.boundary_projection(key)
            self._bdata[key] = torch.as_tensor(g, device=self.device) if g.size else None
        return self._bdata[key]

    def source_data(self, t):
        import torch
        key = float(t)
        if key not in self._src:
            if len(self._src) > 2:
                self._src.clear()
            if getattr(self.tab, "source_zero", False):
                b = None
            elif (getattr(self.tab, "x0", None) is not None and self.tab.ne >= DEVICE_SOURCE_MIN_NE
                  and not getattr(self.tab, "curved", False)):
                # the plan evaluated on the device (source_dev.py, agrees with
                # the numpy restatement to ~1e-16: sin/exp ulps, summation
                # order); small systems keep the restatement, whose cost there
                # is negligible and whose rhs is the reference's to the bit
                if self._devsrc is None:
                    from .source_dev import DeviceSource
                    self._devsrc = DeviceSource(self.tab, self.device)
                b = self._devsrc.load(key)
            else:
                b = self.tab.source_load(key)
            self._src[key] = None if b is None else torch.as_tensor(b, device=self.device)
        return self._src[key]

    def _stream(self):
        return _lib.stream_ptr()

    def _clear_nan(self, *xs):
        """Discard a stale device non-finite flag before a host-API call that
        checks it (a device-path call, e.g. a rejected line-search trial, may
        have left it set)."""
        import torch
        if any(isinstance(x, torch.Tensor) and x.is_cuda for x in xs):
            return
        if self.nl is not None:
            self.nl.reset_bad()
        elif getattr(self, "_h", None) is not None:
            self.lib.ldg_last_bad_element(self._h)

    def _check_nan(self, label):
        if self.nl is not None:
            bad = self.nl.bad_element()
            self.nl.reset_bad()
        else:
            bad = int(self.lib.ldg_last_bad_element(self._h))
        if bad >= 0:
            raise KernelNanError(f"{label} kernel produced non-finite values "
                                 f"(first at element {bad})")

    # -- device operators (torch in / torch out, no host sync) ---------------------------
    def mixed_dev(self, u, t=0.0, homogeneous=False, out=None):
        if self.nl is not None:
            return self.nl.mixed(u, t, homogeneous, out=out)
        q = out if out is not None else self._empty((self.n_elements, self.n_nodes,
                                                     self.ncu, self.nd))
        g = None if homogeneous else self.boundary_data(t)
        _lib.check(self.lib.ldg_compute_mixed(self._h, _lib.ptr(u), _lib.ptr(g),
                                              _lib.ptr(q), self._stream()),
                   "ldg_compute_mixed")
        return q

    def scratch(self, rows=None):
        """Face-export scratch of the fused operator (device, cached); with
        `rows` > n_elements the buffer also holds ghost-element rows."""
        rows = self.n_elements if rows is None else rows
        key = ("x", rows)
        if key not in self._scratch:
            per = int(self.lib.ldg_scratch_doubles(self._h)) // max(self.n_elements, 1)
            self._scratch[key] = self._empty((max(rows * per, 1),))
        return self._scratch[key]

    def operator_pass(self, which, u, tangent, t=0.0, scratch=None, out=None):
        """One pass of the fused operator (1: element pass, 2: completion);
        the partitioned layer exchanges halos between them."""
        R = out if out is not None else self._empty((self.n_elements, self.n_nodes, self.ncu))
        x = scratch if scratch is not None else self.scratch()
        g = None if tangent else self.boundary_data(t)
        b = None if tangent else self.source_data(t)
        _lib.check(self.lib.ldg_operator_pass(self._h, which, int(bool(tangent)), _lib.ptr(u),
                                              _lib.ptr(g), _lib.ptr(b), _lib.ptr(x), _lib.ptr(R),
                                              self._stream()), "ldg_operator_pass")
        return R

    def base_mixed(self, u, t=0.0):
        """q = compute_mixed(u, t) of the tangent's base state, cached per
        (tensor, version, t): the loop-invariant half of every tangent
        (disc.py:602)."""
        if self.kind != "D":
            return None
        # the cache holds the base tensor itself, so its storage cannot be
        # recycled by the allocator for another state with the same address;
        # views of one storage share the version counter
        key = (u.data_ptr(), u._version, tuple(u.shape), float(t))
        if self._baseq is None or self._baseq[0] != key:
            self._baseq = (key, self.nl.mixed(u, t), u)
        return self._baseq[1]

    def residual_dev(self, u, t=0.0, out=None, scratch=None):
        if self.nl is not None:
            return self.nl.residual(u, t, q=self.base_mixed(u, t), out=out)
        R = out if out is not None else self._empty(u.shape)
        x = scratch if scratch is not None else self.scratch()
        _lib.check(self.lib.ldg_residual(
            self._h, _lib.ptr(u), _lib.ptr(self.boundary_data(t)),
            _lib.ptr(self.source_data(t)), _lib.ptr(x), _lib.ptr(R), self._stream()),
            "ldg_residual")
        return R

    def tangent_dev(self, du, out=None, scratch=None, base=None, t=0.0):
        """J(base) du.  The linear fused path ignores `base` and `t` (the
        tangent of a flux linear in (u, q) does not read them)."""
        if self.nl is not None:
            if base is None:
                raise DiscError("the tangent of a nonlinear model needs the base state")
            base = base.reshape(du.shape)
            return self.nl.tangent(base, du, t, q=self.base_mixed(base, t), out=out)
        R = out if out is not None else self._empty(du.shape)
        x = scratch if scratch is not None else self.scratch()
        _lib.check(self.lib.ldg_residual_tangent(self._h, _lib.ptr(du), _lib.ptr(x),
                                                 _lib.ptr(R), self._stream()),
                   "ldg_residual_tangent")
        return R

    def flux_from_mixed_dev(self, u, q, tangent, t=0.0, out=None):
        """The unfused two-kernel structure (mixed -> flux), for comparison."""
        R = out if out is not None else self._empty(u.shape)
        g = None if tangent else self.boundary_data(t)
        b = None if tangent else self.source_data(t)
        _lib.check(self.lib.ldg_flux_from_mixed(self._h, int(bool(tangent)), _lib.ptr(u),
                                                _lib.ptr(q), _lib.ptr(g), _lib.ptr(b),
                                                _lib.ptr(R), self._stream()),
                   "ldg_flux_from_mixed")
        return R

    def mass_apply_dev(self, v, scale=1.0, out=None, base=None, t=0.0):
        if self.nl is not None:
            return self.nl.mass(v, None if base is None else base.reshape(v.shape), t,
                                scale, out=out)
        if not self.tab.mass_const:
            raise DiscError("state-dependent mass is not supported on the B200 path")
        o = out if out is not None else self._empty(v.shape)
        _lib.check(self.lib.ldg_mass_apply(self._h, _lib.ptr(v), float(scale), _lib.ptr(o),
                                           self._stream()), "ldg_mass_apply")
        return o

    def mass_tangent_extra_dev(self, y, du, base, t=0.0, scale=1.0, out=None):
        """(dm/du . du) y (disc.py:927-948); None for a constant mass."""
        if self.mass_is_constant:
            return None
        return self.nl.mass_extra(y, base.reshape(y.shape), du, t, scale, out=out)

    @property
    def mass_is_constant(self):
        if self.nl is not None:
            return bool(self.nl.shape["MASS_CONST"])
        return bool(getattr(self.tab, "mass_const", True))

    def mass_inv_dev(self, v, out=None):
        if self.nl is not None:
            return self.nl.mass_inv(v, out=out)
        o = out if out is not None else self._empty(v.shape)
        _lib.check(self.lib.ldg_mass_inv_apply(self._h, _lib.ptr(v), _lib.ptr(o),
                                               self._stream()), "ldg_mass_inv_apply")
        return o

    # -- chunk-pipelined host calls (fused path) --------------------------------------------
    PIPE_CHUNKS = 12          # measured: 12 -> 4.34, 16 -> 4.32, 24 -> 4.0 GDOF/s e2e

    def _pipe_plan(self):
        """Element chunks and, per chunk, the last chunk holding a face
        neighbour of one of its elements: pass 1 of a chunk needs the input
        rows up to that chunk, pass 2 the exports of pass 1 up to it."""
        if getattr(self, "_pipe", None) is None:
            ne = self.n_elements
            C_ = max(1, min(self.PIPE_CHUNKS, ne // 1024))
            starts = [(ne * c // C_ + 31) // 32 * 32 for c in range(C_)] + [ne]
            starts = [min(x, ne) for x in starts]
            chunk_of = np.searchsorted(np.asarray(starts[1:]), np.arange(ne), side="right")
            nbr = np.where((self.tab.finfo & 3) == 0, self.tab.fnbr, -1)
            far = np.where(nbr >= 0, chunk_of[np.clip(nbr, 0, ne - 1)], 0).max(axis=1)
            dep = np.maximum(np.maximum.reduceat(far, starts[:-1]) if ne else [], np.arange(C_))
            self._pipe = (starts, [int(d) for d in dep])
        return self._pipe

    def _pinned_out(self, shape, as_numpy=False):
        """A pinned host result buffer.  Every call returns a new array as far
        as the caller can tell (disc.py returns fresh arrays): a pooled buffer
        is reused only once the pool holds its last reference, which avoids a
        cudaHostAlloc (~60 ms for 80 MB) per call in a solver loop.  With
        as_numpy the pool holds (tensor, numpy view) pairs and the VIEW is
        what the caller gets and what the reference count is taken of (a
        view does not hold a reference to the tensor object)."""
        import sys
        import torch
        pool = self._scratch.setdefault(("pinned_out", shape, as_numpy), [])
        for i in range(len(pool)):
            obj = pool[i][1] if as_numpy else pool[i]
            if sys.getrefcount(obj) <= 3:        # the pool entry, `obj`, the argument
                return pool[i]
        buf = torch.empty(shape, dtype=torch.float64, pin_memory=True)
        item = (buf, buf.numpy()) if as_numpy else buf
        if len(pool) < 4:
            pool.append(item)
        return item

    def _host_pipeline(self, v, tangent, t):
        """J v or R(v) for a host v through ldg_apply_host_staged: H2D of the
        chunks on a copy stream, the two fused passes per chunk as soon as
        their neighbour rows have arrived, D2H of each finished chunk on a
        second copy stream (PCIe in both directions overlaps the kernels and
        each other).  A pinned torch tensor is sent directly; a numpy array
        (pageable, the reference's convention) is staged chunk by chunk into
        a pinned buffer by the library's host threads, overlapped with the
        transfers.  Returns a pinned torch tensor, or for numpy input a
        numpy view of one (no extra host copy)."""
        import torch
        starts, dep = self._pipe_plan()
        shape = (self.n_elements, self.n_nodes, self.ncu)
        is_np = isinstance(v, np.ndarray)
        if is_np:
            vh = np.ascontiguousarray(v, dtype=np.float64).reshape(shape)
            src, stage = vh.ctypes.data, self._scratch.get(("stage", shape))
            if stage is None:
                stage = self._scratch[("stage", shape)] = torch.empty(
                    shape, dtype=torch.float64, pin_memory=True)
            stage_p = C.c_void_p(stage.data_ptr())
        else:
            vh = v.reshape(shape)
            if not vh.is_pinned():
                vh = vh.pin_memory()
            vh = vh.contiguous()
            src, stage_p = vh.data_ptr(), None
        key = ("pipe", shape)
        if key not in self._scratch:
            self._scratch[key] = (self._empty(shape), self._empty(shape),
                                  np.asarray(starts, dtype=np.int32),
                                  np.asarray(dep, dtype=np.int32))
        vd, R, st_, dp_ = self._scratch[key]
        out = self._pinned_out(tuple(v.shape), as_numpy=is_np)
        out, out_np = out if is_np else (out, None)
        g = None if tangent else self.boundary_data(t)
        b = None if tangent else self.source_data(t)
        _lib.check(self.lib.ldg_apply_host_staged(
            self._h, int(bool(tangent)), C.c_void_p(src), stage_p, C.c_void_p(out.data_ptr()),
            _lib.ptr(vd), _lib.ptr(R), _lib.ptr(self.scratch()), _lib.ptr(g), _lib.ptr(b),
            len(dep), st_.ctypes.data_as(C.c_void_p), dp_.ctypes.data_as(C.c_void_p),
            self._stream()), "ldg_apply_host_staged")
        return out_np if is_np else out

    # -- reference-shaped API ------------------------------------------------------------------
    def _ret(self, x, origin):
        import torch
        if origin == "cuda":
            return x
        if origin == "torch":
            out = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
            out.copy_(x, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            return out
        return x.cpu().numpy()

    def compute_mixed(self, u, t, homogeneous=False):
        """disc.py:436-449."""
        if self.kind != "D":
            raise DiscError("compute_mixed applies to diffusion models")
        self._clear_nan(u)
        ud, dev = self._dev(u)
        q = self.mixed_dev(ud.reshape(self.n_elements, self.n_nodes, self.ncu), t, homogeneous)
        if dev != "cuda":
            self._check_nan("mixed")
        return self._ret(q, dev)

    def _pipelined(self, x):
        import torch
        host = (isinstance(x, np.ndarray) and x.dtype == np.float64) or \
            (isinstance(x, torch.Tensor) and not x.is_cuda)
        return (host and self.nl is None and not self.dense
                and getattr(self, "_h", None) is not None)

    def _packed_host(self, fn, state, *vecs):
        """Run a packed device operator on reference-shaped blocks; returns
        the (u, q, w) blocks like the reference."""
        self._clear_nan(state.u)
        blocks = [self._dev(b)[0] if b is not None else None for b in
                  (state.u, state.q, state.w)]
        dev = self._dev(state.u)[1]
        Y = self._cat([b for b in blocks if b is not None])
        args = []
        for v in vecs:
            vb = [self._dev(b)[0] if b is not None else None for b in v]
            args.append(self._cat([b for b in vb if b is not None]))
        out = fn(*args, Y)
        self._check_nan("flux")
        u, q, w = self.unpack(out)
        return (self._ret(u, dev), None if q is None else self._ret(q, dev),
                None if w is None else self._ret(w, dev))

    def residual(self, state):
        """disc.py:588-589 -> (Ru, Rq, Rw)."""
        self._clear_nan(state.u)
        if self.nl is not None and self.multi_block:
            return self._packed_host(lambda Y: self.residual_packed_dev(Y, state.t), state)
        if self._pipelined(state.u):
            R = self._host_pipeline(state.u, False, state.t)
            self._check_nan("flux")
            return R, None, None
        ud, dev = self._dev(state.u)
        R = self.residual_dev(ud.reshape(self.n_elements, self.n_nodes, self.ncu), state.t)
        if dev != "cuda":
            self._check_nan("flux")
        return self._ret(R, dev), None, None

    def residual_tangent(self, state, du, dq=None, dw=None):
        """disc.py:591-593 (the reference linearisation)."""
        self._clear_nan(du)
        if self.nl is not None and self.multi_block:
            return self._packed_host(lambda V, Y: self.tangent_packed_dev(V, Y, state.t),
                                     state, (du, dq, dw))
        if self._pipelined(du):
            R = self._host_pipeline(du, True, state.t)
            self._check_nan("flux")
            return R, None, None
        dd, dev = self._dev(du)
        shape = (self.n_elements, self.n_nodes, self.ncu)
        base = None
        if self.nl is not None:
            base = self._dev(state.u)[0].reshape(shape)
        R = self.tangent_dev(dd.reshape(shape), base=base, t=state.t)
        if dev != "cuda":
            self._check_nan("flux")
        return self._ret(R, dev), None, None

    def mass_apply(self, state, vu, vq=None, vw=None):
        """disc.py:897-925."""
        self._clear_nan(vu)
        if self.nl is not None and self.multi_block:
            return self._packed_host(lambda V, Y: self.mass_packed_dev(V, Y, state.t),
                                     state, (vu, vq, vw))
        vd, dev = self._dev(vu)
        shape = (self.n_elements, self.n_nodes, self.ncu)
        base = None if self.mass_is_constant else self._dev(state.u)[0].reshape(shape)
        M = self.mass_apply_dev(vd.reshape(shape), base=base, t=state.t)
        if dev != "cuda" and self.nl is not None:
            self._check_nan("mass")
        return self._ret(M, dev), None, None

    def mass_tangent_extra(self, state, y_u, du, dq=None, dw=None):
        """disc.py:927-948: None for a constant mass."""
        if self.mass_is_constant:
            return None
        shape = (self.n_elements, self.n_nodes, self.ncu)
        yd, dev = self._dev(y_u)
        out = self.mass_tangent_extra_dev(yd.reshape(shape), self._dev(du)[0].reshape(shape),
                                          self._dev(state.u)[0].reshape(shape), state.t)
        return self._ret(out, dev)

    # -- packed multi-block operators (kind W / ODE blocks; generated path) ------------------
    def _blocks_dev(self, Y):
        return self.unpack(Y)

    def _cat(self, parts):
        import torch
        return torch.cat([p.reshape(-1) for p in parts if p is not None])

    def residual_packed_dev(self, Y, t=0.0):
        """[Ru | Rq | Rw] of a packed device state (disc.py:595-653, 866-893)."""
        u, q, w = self._blocks_dev(Y)
        qq = self.base_mixed(u, t) if self.kind == "D" else q
        Ru = self.nl.residual(u, t, q=qq, w=w)
        Rq = self.nl.gradient_residual(u, q, t) if self.kind == "W" else None
        Rw = self.nl.ode(u, qq, w, t) if self.nw > 0 else None
        return self._cat([Ru, Rq, Rw])

    def tangent_packed_dev(self, V, Y, t=0.0):
        """The reference linearisation on packed vectors."""
        u, q, w = self._blocks_dev(Y)
        du, dq, dw = self._blocks_dev(V)
        qq, dqq = q, dq
        if self.kind == "D":
            qq = self.base_mixed(u, t)
            dqq = self.nl.mixed(du, t, homogeneous=True) if self.nw > 0 else None
        dRu = self.nl.tangent(u, du, t, q=qq, w=w, dq=dq, dw=dw)
        dRq = self.nl.gradient_residual(du, dq, t, tangent=True) if self.kind == "W" else None
        dRw = self.nl.ode(u, qq, w, t, du=du, dq=dqq, dw=dw) if self.nw > 0 else None
        return self._cat([dRu, dRq, dRw])

    def mass_packed_dev(self, V, Y, t=0.0, scale=1.0):
        """[M(u) vu | M vq | alpha vw] (disc.py:897-925)."""
        u, _, _ = self._blocks_dev(Y)
        vu, vq, vw = self._blocks_dev(V)
        Mu = self.nl.mass(vu, u, t, scale)
        Mq = self.nl.mass_q(vq, scale) if self.kind == "W" else None
        Mw = (scale * self.model.ode.alpha) * vw if self.nw > 0 else None
        return self._cat([Mu, Mq, Mw])

    def mass_extra_packed_dev(self, Yd, V, Y, t=0.0, scale=1.0):
        """(dm/du du) y on the u block, zero elsewhere (disc.py:927-948)."""
        import torch
        if self.mass_is_constant:
            return None
        u, _, _ = self._blocks_dev(Y)
        du, _, _ = self._blocks_dev(V)
        yu, _, _ = self._blocks_dev(Yd)
        out = torch.zeros_like(V)
        out[: u.numel()].copy_(self.nl.mass_extra(yu, u, du, t, scale).reshape(-1))
        return out

    def mass_inv_packed_dev(self, V):
        """MassPreconditioner.apply on packed vectors (driver.py:99-106)."""
        vu, vq, vw = self._blocks_dev(V)
        return self._cat([self.nl.mass_inv(vu),
                          self.nl.mass_inv_q(vq) if self.kind == "W" else None,
                          vw / self.model.ode.alpha if self.nw > 0 else None])

    def interpolate_initial(self):
        """disc.py:420-432 (host evaluation of the init plan at the nodes)."""
        from .expr import evaluate
        x = self.disc.node_x
        b = {"t": 0.0, **self.model.mu_bindings()}
        for k in range(self.nd):
            b[f"x{k + 1}"] = x[..., k].ravel()
        v = evaluate(self.model.init_plan(), b)
        if not np.isfinite(v).all():
            col = int(np.argwhere(~np.isfinite(v))[0][1])
            raise KernelNanError("initial kernel produced non-finite values "
                                 f"(first at element {col // self.n_nodes})")
        B = self.n_elements * self.n_nodes
        if v.shape[1] != B:
            v = np.broadcast_to(v, (v.shape[0], B))
        vals = np.moveaxis(v.reshape((v.shape[0], self.n_elements, self.n_nodes)), 0, -1)
        k = self.ncu
        u = np.ascontiguousarray(vals[..., :k])
        q = w = None
        if self.kind == "W":
            q = np.ascontiguousarray(vals[..., k:k + self.ncu * self.nd]).reshape(
                self.n_elements, self.n_nodes, self.ncu, self.nd)
            k += self.ncu * self.nd
        if self.nw > 0:
            w = np.ascontiguousarray(vals[..., k:k + self.nw])
        return SolverState(u=u, q=q, w=w, t=0.0)

    def interpolate_initial_dev(self):
        """interpolate_initial with the init plan evaluated on the device at
        every node (source_dev.device_initial_values): device u / q / w, no
        host pass over the nodes."""
        from .source_dev import device_initial_values
        v = device_initial_values(self.tab, self.model, self.device)
        k = self.ncu
        u = v[..., :k].contiguous()
        q = w = None
        if self.kind == "W":
            q = v[..., k:k + self.ncu * self.nd].contiguous().reshape(
                self.n_elements, self.n_nodes, self.ncu, self.nd)
            k += self.ncu * self.nd
        if self.nw > 0:
            w = v[..., k:k + self.nw].contiguous()
        return SolverState(u=u, q=q, w=w, t=0.0)
