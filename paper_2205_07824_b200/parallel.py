"""Element-partitioned multi-GPU layer.

One process per GPU.  Each rank owns a contiguous range of global elements
(x-slabs on the structured meshes, whose elements are numbered x-outermost,
mesh.py:156-163); the global face tables are built once (bit-exact with the
reference) and sliced, so connectivity, switch bits and gather indices of
every partition are the global ones.  Per operator application two halo
steps exchange ghost-element data over NCCL (gloo on CPU in the tests):

  1. before pass 1: the state of the ghost elements (neighbours owned by
     other ranks) -- the u^ / penalty gathers read their face nodes;
  2. between pass 1 and pass 2: the ghost elements' face exports
     X = sJ n.(Aq q), which carry the neighbour share of f(., q^).

Krylov reductions are allreduced sums of per-rank partials
(:class:`DistVecOps`).  Ranks are on one node: NCCL runs over NVLink 5 /
NVSwitch.
"""

from __future__ import annotations

import numpy as np

from .tables import DiscError


def element_ranges(ne, nranks):
    """Balanced contiguous element ranges [e0, e1) per rank."""
    base, rem = divmod(ne, nranks)
    starts = np.cumsum([0] + [base + (1 if r < rem else 0) for r in range(nranks)])
    return [(int(starts[r]), int(starts[r + 1])) for r in range(nranks)]


class PartitionPlan:
    """Local numbering, sliced tables and halo lists of one rank."""

    def __init__(self, tab, nranks, rank):
        self.nranks, self.rank = nranks, rank
        ne = tab.ne
        self.ranges = element_ranges(ne, nranks)
        e0, e1 = self.ranges[rank]
        self.e0, self.e1 = e0, e1
        self.ne_loc = e1 - e0
        owner = np.zeros(ne, dtype=np.int64)
        for r, (a, b) in enumerate(self.ranges):
            owner[a:b] = r
        self.owner = owner
        fnbr = tab.fnbr[e0:e1].astype(np.int64)
        finfo = tab.finfo[e0:e1]
        interior = (finfo & 3) == 0
        nbrs = np.where(interior, fnbr, -1)
        ext = np.unique(nbrs[(nbrs >= 0) & ((nbrs < e0) | (nbrs >= e1))])
        self.ghosts = ext                                 # global ids, sorted
        self.n_ghost = ext.size
        g2l = {int(g): self.ne_loc + k for k, g in enumerate(ext.tolist())}
        loc = np.where(interior & (nbrs >= e0) & (nbrs < e1), nbrs - e0, -1)
        ghost_mask = interior & ((nbrs < e0) | (nbrs >= e1))
        if ghost_mask.any():
            loc[ghost_mask] = np.searchsorted(ext, nbrs[ghost_mask]) + self.ne_loc
        # boundary rows referenced by owned elements -> local rows
        bmask = ~interior
        brows = np.unique(fnbr[bmask]) if bmask.any() else np.zeros(0, np.int64)
        self.brows = brows
        if bmask.any():
            loc[bmask] = np.searchsorted(brows, fnbr[bmask])
        self.fnbr = loc.astype(np.int32)
        self.finfo = finfo.copy()
        self.ftau = tab.ftau[e0:e1].copy()
        self.geo = tab.geo[e0:e1].copy()
        del g2l
        # halo lists: what I send to q = my owned elements adjacent to q's range
        self.recv = {}
        self.send = {}
        for q in range(nranks):
            if q == rank:
                continue
            mine = self.ghosts[owner[self.ghosts] == q]
            if mine.size:
                self.recv[q] = (np.searchsorted(self.ghosts, mine) + self.ne_loc).astype(np.int64)
            adj = (owner[np.where(nbrs >= 0, nbrs, 0)] == q) & (nbrs >= 0)
            rows = np.nonzero(adj.any(axis=1))[0]
            if rows.size:
                self.send[q] = rows.astype(np.int64)          # local owned rows, sorted
        if np.any(self.fnbr < 0):
            raise DiscError("partition left an unresolved neighbour")


class LocalTables:
    """TensorTables interface over one partition (rows sliced, neighbours
    renumbered to [owned | ghosts])."""

    def __init__(self, tab, plan):
        self._g, self.plan = tab, plan
        for k in ("nd", "n1", "ncu", "nf", "nfn", "p", "nmap", "d1", "m1", "s1", "clo", "chi",
                  "m1inv", "au", "aq", "flux_uses_u", "mass_coef", "mass_const", "source_zero",
                  "model", "master", "mesh", "topo", "bc_groups"):
            setattr(self, k, getattr(tab, k, None))     # (generated-path tables lack au/aq)
        e0, e1 = plan.e0, plan.e1
        self.ne = plan.ne_loc
        self.geo, self.fnbr, self.finfo, self.ftau = plan.geo, plan.fnbr, plan.finfo, plan.ftau
        self.detj, self.invjt = tab.detj[e0:e1], tab.invjt[e0:e1]
        self.J, self.x0 = tab.J[e0:e1], tab.x0[e0:e1]
        self.elem_vol = tab.elem_vol[e0:e1]
        self.switch = tab.switch          # global face bits (for reference)
        self.fi_h, self.fb_h = tab.fi_h, tab.fb_h

    def node_coords(self, elems=None, nodes=None):
        e = np.arange(self.plan.e0, self.plan.e1) if elems is None else \
            np.asarray(elems) + self.plan.e0
        return self._g.node_coords(e, nodes)

    def face_node_vol(self, lf):
        return self._g.face_node_vol(lf)

    def boundary_projection(self, t):
        g = self._g.boundary_projection(t)
        return g[self.plan.brows] if g.size else g

    def source_load(self, t):
        b = self._g.source_load(t)
        return None if b is None else b[self.plan.e0:self.plan.e1]


class HaloExchanger:
    """Ghost-row exchange of an (n_owned + n_ghost, width) array with
    torch.distributed point-to-point ops (NCCL on GPU, gloo on CPU)."""

    def __init__(self, plan, group=None):
        self.plan, self.group = plan, group
        self._idx = {}

    def _rows(self, kind, q, rows, device):
        key = (kind, q, str(device))
        if key not in self._idx:                 # index rows uploaded once per peer
            import torch
            self._idx[key] = torch.as_tensor(rows, device=device)
        return self._idx[key]

    def exchange(self, arr):
        import torch
        import torch.distributed as dist
        # gloo moves host memory only: stage device buffers through the host
        # (testing several ranks on one GPU); NCCL sends device buffers directly
        stage = arr.is_cuda and dist.get_backend(self.group) == "gloo"
        ops, recv_bufs = [], []
        flat = arr.reshape(arr.shape[0], -1)
        for q, rows in sorted(self.plan.send.items()):
            idx = self._rows("s", q, rows, arr.device)
            buf = flat.index_select(0, idx).contiguous()
            if stage:
                buf = buf.cpu()
            ops.append(dist.P2POp(dist.isend, buf, q, group=self.group))
        for q, rows in sorted(self.plan.recv.items()):
            buf = torch.empty((rows.size, flat.shape[1]), dtype=arr.dtype,
                              device="cpu" if stage else arr.device)
            recv_bufs.append((self._rows("r", q, rows, arr.device), buf))
            ops.append(dist.P2POp(dist.irecv, buf, q, group=self.group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        for idx, buf in recv_bufs:
            flat.index_copy_(0, idx, buf.to(arr.device))
        return arr


class DistVecOps:
    """VecOps with every reduction allreduced over the process group (sum
    of per-rank partials; norms from allreduced squares)."""

    def __init__(self, base, group=None):
        self.b, self.group = base, group

    def _ar(self, t):
        import torch.distributed as dist
        if t.is_cuda and dist.get_backend(self.group) == "gloo":
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def dot(self, x, y, out):
        self.b.dot(x, y, out)
        self._ar(out)

    def nrm2(self, x, out):
        self.b.dot(x, x, out)
        self._ar(out)
        out.sqrt_()

    def norm(self, x):
        out = x.new_zeros(1)
        self.nrm2(x, out)
        return float(out.item())

    def amax(self, x):
        """Global max |x_i| (fd_epsilon's ||base||_inf, solver.py:187)."""
        import torch
        import torch.distributed as dist
        m = x.abs().max().reshape(1) if x.numel() else x.new_zeros(1)
        m = torch.where(torch.isnan(m), torch.full_like(m, float("inf")), m)
        if m.is_cuda and dist.get_backend(self.group) == "gloo":
            h = m.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.MAX, group=self.group)
            m.copy_(h)
        else:
            dist.all_reduce(m, op=dist.ReduceOp.MAX, group=self.group)
        return float(m.item())

    def axpy(self, *a, **k):
        return self.b.axpy(*a, **k)

    def div(self, *a, **k):
        return self.b.div(*a, **k)

    def mgs_step(self, vi, h_in, w, vnext, h_out):
        self.b.mgs_step(vi, h_in, w, vnext, h_out)
        if vnext is not None:
            self._ar(h_out)

    def cgs_dots(self, V, k, w, h):
        self.b.cgs_dots(V, k, w, h)
        self._ar(h[:k])

    def cgs_update(self, V, k, h, w, nrm_out):
        self.b.cgs_update(V, k, h, w, None)
        self.nrm2(w, nrm_out)

    def dcgs_dots(self, V, k, x, y, hx, hy):
        self.b.dcgs_dots(V, k, x, y, hx, hy)
        self._ar(hx[:k])
        self._ar(hy[:k])

    def dcgs_update(self, V, m, s, t, v, w, out, inv_alpha, gamma, nrm_out):
        self.b.dcgs_update(V, m, s, t, v, w, out, inv_alpha, gamma, None)
        self.nrm2(out, nrm_out)

    def combine(self, *a, **k):
        return self.b.combine(*a, **k)


class PartitionedLdgSystem:
    """One rank's share of the LDG operator on its GPU: owned elements plus a
    ghost layer, native fused passes, halo exchanges in between.

    ``exchange(arr)`` fills the ghost rows of an (owned + ghost, ...) array;
    the default is the NCCL/gloo :class:`HaloExchanger`.  Vectors handed to
    ``residual_dev`` / ``tangent_dev`` hold the owned elements only.
    """

    def __init__(self, model, mesh, topology, master, nranks, rank, device=None,
                 exchanger=None, tables=None):
        import torch
        from .system import LdgSystem
        from .tables import TensorTables
        gtab = tables if tables is not None else TensorTables(model, mesh, topology, master)
        self.plan = PartitionPlan(gtab, nranks, rank)
        self.local = LocalTables(gtab, self.plan)
        self.sys = LdgSystem(model, mesh, topology, master, device=device, tables=self.local)
        # exports stay in the producer's rows: those rows are what the halo
        # exchange ships to the ranks holding the element as a ghost
        from . import _lib as L
        L.check(self.sys.lib.ldg_set_export_layout(self.sys._h, 0), "ldg_set_export_layout")
        self.exchanger = exchanger if exchanger is not None else HaloExchanger(self.plan)
        p = self.plan
        self.n_elements, self.n_nodes, self.ncu = p.ne_loc, master.n_nodes, model.ncu
        self.n_dofs = p.ne_loc * master.n_nodes * model.ncu
        self.kind, self.model, self.device = model.kind, model, self.sys.device
        self.u_ext = torch.zeros((p.ne_loc + p.n_ghost, master.n_nodes, model.ncu),
                                 dtype=torch.float64, device=self.sys.device)
        self.X = self.sys.scratch(rows=p.ne_loc + p.n_ghost)

    def apply(self, u, tangent, t=0.0, out=None, exchange=True):
        p = self.plan
        self.u_ext[:p.ne_loc].copy_(u.reshape(p.ne_loc, self.n_nodes, self.ncu))
        if exchange:
            self.exchanger.exchange(self.u_ext)
        R = self.sys.operator_pass(1, self.u_ext, tangent, t, scratch=self.X, out=out)
        if exchange:
            self.exchange_exports()
        return self.sys.operator_pass(2, self.u_ext, tangent, t, scratch=self.X, out=R)

    def exchange_exports(self):
        p = self.plan
        per = self.X.numel() // (p.ne_loc + p.n_ghost)
        self.exchanger.exchange(self.X[: (p.ne_loc + p.n_ghost) * per].view(-1, per))

    def residual_dev(self, u, t=0.0, out=None):
        return self.apply(u, False, t, out)

    def tangent_dev(self, du, out=None, base=None, t=0.0):
        """Linear fused operator: the tangent reads neither base nor t."""
        return self.apply(du, True, 0.0, out)


class LocalBus:
    """Single-process stand-in for the halo exchange among R partitions
    living on one GPU (partition and halo logic testable without
    8 GPUs): ghost rows are copied device-to-device from the owners."""

    def __init__(self, parts):
        self.parts = parts

    def fill(self, getter):
        import torch
        for p in self.parts:
            plan = p.plan
            arr = getter(p)
            flat = arr.reshape(arr.shape[0], -1)
            for k, g in enumerate(plan.ghosts.tolist()):
                q = int(plan.owner[g])
                src = getter(self.parts[q])
                flat[plan.ne_loc + k].copy_(src.reshape(src.shape[0], -1)[g - self.parts[q].plan.e0])
        del torch

    def apply_all(self, us, tangent, t=0.0):
        """Operator on every partition in lockstep (pass 1 -> exports -> pass 2)."""
        for p, u in zip(self.parts, us):
            p.u_ext[:p.plan.ne_loc].copy_(u.reshape(p.plan.ne_loc, p.n_nodes, p.ncu))
        self.fill(lambda p: p.u_ext)
        Rs = [p.sys.operator_pass(1, p.u_ext, tangent, t, scratch=p.X) for p in self.parts]
        per = [p.X.numel() // (p.plan.ne_loc + p.plan.n_ghost) for p in self.parts]
        self.fill(lambda p: p.X[: (p.plan.ne_loc + p.plan.n_ghost) * per[self.parts.index(p)]]
                  .view(-1, per[self.parts.index(p)]))
        return [p.sys.operator_pass(2, p.u_ext, tangent, t, scratch=p.X, out=R)
                for p, R in zip(self.parts, Rs)]


# ---------------------------------------------------------------------------
# generated-kernel (nonlinear / kind C) models
# ---------------------------------------------------------------------------


class LocalNlTables(LocalTables):
    """NlTables interface over one partition: the affine maps and
    element-face geometry sliced, boundary data restricted to the
    partition's boundary rows."""

    def __init__(self, tab, plan):
        super().__init__(tab, plan)
        for k in ("nq1", "fxi", "fw", "periodic", "nonlinear", "tau_i", "tau_b"):
            setattr(self, k, getattr(tab, k))
        e0, e1 = plan.e0, plan.e1
        self.xmap = tab.xmap[e0:e1]
        self.fgeo = tab.fgeo[e0:e1]
        self.n_boundary = int(plan.brows.size)

    def boundary_points(self, t):
        g = self._g.boundary_points(t)
        return g[self.plan.brows] if g.size else g


class PartitionedNlSystem:
    """One rank's share of a generated-kernel model: owned elements plus a
    ghost layer.  Per residual: the ghost u rows (halo 1), the owned mixed
    gradient, its ghost rows (halo 2, kind D), then the element kernel.  The
    tangent exchanges the direction the same way; the base state's ghost u / q
    are exchanged once per base (cached like the single-GPU base q)."""

    def __init__(self, model, mesh, topology, master, nranks, rank, device=None,
                 exchanger=None, tables=None):
        import torch
        from .nonlinear import NlOperator, NlTables
        gtab = tables if tables is not None else NlTables(model, mesh, topology, master)
        self.plan = PartitionPlan(gtab, nranks, rank)
        self.local = LocalNlTables(gtab, self.plan)
        self.device = torch.device(device if device is not None else "cuda")
        self.nl = NlOperator(self.local, self.device)
        self.exchanger = exchanger if exchanger is not None else HaloExchanger(self.plan)
        p = self.plan
        self.model, self.kind = model, model.kind
        self.n_elements, self.n_nodes, self.ncu = p.ne_loc, master.n_nodes, model.ncu
        self.nd = mesh.nd
        self.n_dofs = p.ne_loc * master.n_nodes * model.ncu
        rows = p.ne_loc + p.n_ghost
        self._ushape = (rows, master.n_nodes, model.ncu)
        self._qshape = (rows, master.n_nodes, model.ncu, mesh.nd)
        self._base = None

    def _new(self, shape):
        import torch
        return torch.zeros(shape, dtype=torch.float64, device=self.device)

    def _exchange(self, arr):
        if self.exchanger:
            self.exchanger.exchange(arr)

    def extend(self, u):
        """(owned) -> (owned + ghost) rows with the halo filled."""
        ext = self._new(self._ushape)
        ext[: self.plan.ne_loc].copy_(u.reshape(self.plan.ne_loc, self.n_nodes, self.ncu))
        self._exchange(ext)
        return ext

    def mixed_ext(self, u_ext, t, homogeneous=False):
        q = self._new(self._qshape)
        self.nl.mixed(u_ext, t, homogeneous, out=q[: self.plan.ne_loc])
        self._exchange(q)
        return q

    def base_ext(self, base, t):
        key = (base.data_ptr(), base._version, float(t))
        if self._base is None or self._base[0] != key:
            ue = self.extend(base)
            qe = self.mixed_ext(ue, t) if self.kind == "D" else None
            self._base = (key, ue, qe, base)
        return self._base[1], self._base[2]

    def residual_dev(self, u, t=0.0, out=None):
        ue, qe = self.base_ext(u, t)
        R = self.nl.residual(ue, t, q=qe)
        return R[: self.plan.ne_loc] if out is None else out.copy_(R[: self.plan.ne_loc])

    def tangent_dev(self, du, out=None, base=None, t=0.0):
        ue, qe = self.base_ext(base, t)
        de = self.extend(du)
        dq = self.mixed_ext(de, t, homogeneous=True) if self.kind == "D" else None
        R = self.nl.tangent(ue, de, t, q=qe, dq=dq)
        return R[: self.plan.ne_loc] if out is None else out.copy_(R[: self.plan.ne_loc])


def nl_apply_all(parts, us, tangent, bases=None, t=0.0):
    """Single-process lockstep of R partitions of a generated-kernel model on
    one GPU (ghost rows by device copies): the two halo steps of
    PartitionedNlSystem with a LocalBus in place of NCCL."""
    bus = LocalBus(parts)
    n = len(parts)

    def ext(vals):
        arrs = []
        for p, v in zip(parts, vals):
            a = p._new(p._ushape)
            a[: p.plan.ne_loc].copy_(v.reshape(p.plan.ne_loc, p.n_nodes, p.ncu))
            arrs.append(a)
        bus.fill(lambda p: arrs[parts.index(p)])
        return arrs

    def mixed(arrs, homogeneous):
        if parts[0].kind != "D":
            return [None] * n
        qs = []
        for p, a in zip(parts, arrs):
            q = p._new(p._qshape)
            p.nl.mixed(a, t, homogeneous, out=q[: p.plan.ne_loc])
            qs.append(q)
        bus.fill(lambda p: qs[parts.index(p)].reshape(qs[parts.index(p)].shape[0], -1))
        return qs

    base = ext(bases if bases is not None else us)
    qb = mixed(base, False)
    if not tangent:
        return [p.nl.residual(a, t, q=q)[: p.plan.ne_loc] for p, a, q in zip(parts, base, qb)]
    d = ext(us)
    dq = mixed(d, True)
    return [p.nl.tangent(a, b, t, q=q, dq=dd)[: p.plan.ne_loc]
            for p, a, b, q, dd in zip(parts, base, d, qb, dq)]
