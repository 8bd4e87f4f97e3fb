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
        if hasattr(tab, "nmap"):          # tensor tables: face-node halos
            self._face_halo(tab)
        else:                             # simplex tables: whole ghost rows
            self.interior = (0, 0)
            self.row_send = {q: r for q, r in self.send.items()}
            self.row_recv = {q: r - self.ne_loc for q, r in self.recv.items()}

    def _cut_pairs(self, tab, recv_rank, send_rank):
        """Cut (element, face) slots of recv_rank's elements whose neighbour
        send_rank owns, as (neighbour global id, neighbour volume nodes read,
        neighbour local face) -- computed identically on both sides from the
        global tables, so the send and receive orders agree."""
        a, b = self.ranges[recv_rank]
        info = tab.finfo[a:b]
        nbr = tab.fnbr[a:b].astype(np.int64)
        interior = (info & 3) == 0
        cut = interior & (self.owner[np.where(interior, nbr, 0)] == send_rank) & \
            ((nbr < a) | (nbr >= b))
        el, lf = np.nonzero(cut)
        g = nbr[el, lf]
        mid = (info[el, lf] >> 8) & 0xffff
        nlf = (info[el, lf] >> 4) & 7
        return g, np.asarray(tab.nmap)[mid], nlf

    def _face_halo(self, tab):
        """Face-node halo lists: per peer, only the neighbour
        face nodes the cut faces read (n1^(nd-1) per face instead of the
        whole n1^nd element row) and only the export slot of the face that
        faces this rank (one of 2 nd).  Flat row indices:
          u_recv[q]: rows of u_ghost viewed (n_ghost * nb, ncu)
          u_send[q]: rows of the owned u viewed (ne_loc * nb, ncu)
          x_recv[q] / x_send[q]: rows of X viewed (rows * 2nd, nfn * ncu)."""
        nb = int(tab.n1) ** int(tab.nd)
        nf = int(tab.nf)
        self.nb, self.nf = nb, nf
        self.u_recv, self.u_send, self.x_recv, self.x_send = {}, {}, {}, {}
        me = self.rank
        for q in range(self.nranks):
            if q == me:
                continue
            for recv_rank, send_rank, own in ((me, q, False), (q, me, True)):
                g, nodes, nlf = self._cut_pairs(tab, recv_rank, send_rank)
                if g.size == 0:
                    continue
                un = np.unique(g[:, None] * nb + nodes)             # (element, node) keys
                xk = np.unique(g * nf + nlf)                          # (element, face) keys
                if own:                  # I send: rows of my owned arrays
                    self.u_send[q] = un - self.e0 * nb
                    self.x_send[q] = xk - self.e0 * nf
                else:                    # I receive: rows of my ghost arrays
                    gk = np.searchsorted(self.ghosts, un // nb)
                    self.u_recv[q] = gk * nb + un % nb
                    xg = np.searchsorted(self.ghosts, xk // nf)
                    self.x_recv[q] = (self.ne_loc + xg) * nf + xk % nf
        # owned elements with a ghost neighbour; when they sit at the two ends
        # of the range (x-slabs) [a, b) is the interior, computed while the
        # halos are in flight
        touch = (np.where((self.finfo & 3) == 0, self.fnbr, -1) >= self.ne_loc).any(axis=1)
        idx = np.nonzero(touch)[0]
        a = 0
        while a < self.ne_loc and touch[a]:
            a += 1
        b = self.ne_loc
        while b > a and touch[b - 1]:
            b -= 1
        if touch[a:b].any():                  # boundary elements inside: no overlap
            a = b = 0
        self.interior = (a, b)
        self.n_boundary = int(idx.size)


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


class _Pending:
    """In-flight list exchange: wait() completes the receives and scatters
    them into the destination (on the current stream for NCCL)."""

    def __init__(self, works, recv_bufs, dst, stage):
        self.works, self.recv_bufs, self.dst, self.stage = works, recv_bufs, dst, stage

    def wait(self):
        for w in self.works:
            w.wait()
        for idx, buf in self.recv_bufs:
            self.dst.index_copy_(0, idx, buf.to(self.dst.device) if self.stage else buf)
        self.works = []


class FaceHaloExchanger(HaloExchanger):
    """Face-node halos (PartitionPlan.u_send / u_recv, x_send / x_recv):
    rows gathered from a flat source, sent with batched NCCL point-to-point
    ops, scattered into a flat destination on wait().  start() returns at
    once on NCCL (the transfer runs on NCCL's stream while the caller
    launches interior work); gloo (CPU tests, ranks sharing one GPU) stages
    through the host and completes before returning."""

    def start(self, src, dst, send, recv):
        import torch
        import torch.distributed as dist
        stage = src.is_cuda and dist.get_backend(self.group) == "gloo"
        ops, recv_bufs = [], []
        for q, rows in sorted(send.items()):
            buf = src.index_select(0, self._rows(("s", id(send)), q, rows, src.device))
            ops.append(dist.P2POp(dist.isend, buf.cpu() if stage else buf, q, group=self.group))
        for q, rows in sorted(recv.items()):
            buf = torch.empty((rows.size,) + tuple(dst.shape[1:]), dtype=dst.dtype,
                              device="cpu" if stage else dst.device)
            recv_bufs.append((self._rows(("r", id(recv)), q, rows, dst.device), buf))
            ops.append(dist.P2POp(dist.irecv, buf, q, group=self.group))
        works = dist.batch_isend_irecv(ops) if ops else []
        p = _Pending(works, recv_bufs, dst, stage)
        if stage:
            p.wait()
        return p


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

    def div_guarded(self, *a, **k):
        return self.b.div_guarded(*a, **k)

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
        """Both dot sweeps' partials in ONE allreduce (hx, hy side by side
        in a scratch row)."""
        import torch
        self.b.dcgs_dots(V, k, x, y, hx, hy)
        buf = getattr(self, "_dd", None)
        if buf is None or buf.numel() < 2 * k or buf.device != hx.device:
            buf = self._dd = torch.empty(2 * max(k, 256), dtype=hx.dtype, device=hx.device)
        buf[:k].copy_(hx[:k])
        buf[k:2 * k].copy_(hy[:k])
        self._ar(buf[:2 * k])
        hx[:k].copy_(buf[:k])
        hy[:k].copy_(buf[k:2 * k])

    def dcgs_update(self, V, m, s, t, v, w, out, inv_alpha, gamma, nrm_out):
        self.b.dcgs_update(V, m, s, t, v, w, out, inv_alpha, gamma, None)
        self.nrm2(out, nrm_out)

    def combine(self, *a, **k):
        return self.b.combine(*a, **k)


class PartitionedLdgSystem:
    """One rank's share of the LDG operator on its GPU: owned elements plus a
    ghost layer, native fused passes, face-node halo exchanges in between.

    The owned vector is used in place: neighbour rows >= n_owned are read
    from the ghost buffer ``u_ghost`` (``ldg_set_ghost_rows``), which holds
    only the face nodes the cut faces read.  Per operator application
    (``apply``), with [a, b) the owned elements that touch no ghost:

      start u halo      | pass 1 on [a, b)        (overlapped)
      wait; pass 1 on the rest
      start export halo | pass 2 on [a, b)        (overlapped)
      wait; pass 2 on the rest

    ``exchanger=False`` leaves the halos to the caller (:class:`LocalBus`).
    Vectors handed to ``residual_dev`` / ``tangent_dev`` hold the owned
    elements only.
    """

    def __init__(self, model, mesh, topology, master, nranks, rank, device=None,
                 exchanger=None, tables=None):
        import torch
        from .system import LdgSystem
        from .tables import TensorTables
        from . import _lib as L
        gtab = tables if tables is not None else TensorTables(model, mesh, topology, master)
        self.plan = PartitionPlan(gtab, nranks, rank)
        self.local = LocalTables(gtab, self.plan)
        self.sys = LdgSystem(model, mesh, topology, master, device=device, tables=self.local)
        # exports stay in the producer's rows: those rows are what the halo
        # exchange ships to the ranks holding the element as a ghost
        L.check(self.sys.lib.ldg_set_export_layout(self.sys._h, 0), "ldg_set_export_layout")
        self.exchanger = exchanger if exchanger is not None else FaceHaloExchanger(self.plan)
        p = self.plan
        self.n_elements, self.n_nodes, self.ncu = p.ne_loc, master.n_nodes, model.ncu
        self.n_dofs = p.ne_loc * master.n_nodes * model.ncu
        self.kind, self.model, self.device = model.kind, model, self.sys.device
        self.u_ghost = torch.zeros((max(p.n_ghost, 1), master.n_nodes, model.ncu),
                                   dtype=torch.float64, device=self.sys.device)
        L.check(self.sys.lib.ldg_set_ghost_rows(self.sys._h, p.ne_loc, L.ptr(self.u_ghost)),
                "ldg_set_ghost_rows")
        self.X = self.sys.scratch(rows=p.ne_loc + p.n_ghost)
        self._xper = self.X.numel() // (p.ne_loc + p.n_ghost)

    def x_rows(self):
        """The export scratch viewed (rows * 2nd, nfn * ncu): one row per
        element face slot."""
        p = self.plan
        return self.X[: (p.ne_loc + p.n_ghost) * self._xper].view(
            (p.ne_loc + p.n_ghost) * p.nf, self._xper // p.nf)

    def start_u_halo(self, u):
        p = self.plan
        return self.exchanger.start(u.reshape(p.ne_loc * p.nb, self.ncu),
                                    self.u_ghost.view(-1, self.ncu), p.u_send, p.u_recv)

    def start_x_halo(self):
        xr = self.x_rows()
        return self.exchanger.start(xr, xr, self.plan.x_send, self.plan.x_recv)

    def _pass(self, which, u, tangent, t, R, e0, e1):
        from . import _lib as L
        if e1 <= e0:
            return
        g = None if tangent else self.sys.boundary_data(t)
        b = None if tangent else self.sys.source_data(t)
        L.check(self.sys.lib.ldg_operator_pass_range(
            self.sys._h, which, int(bool(tangent)), L.ptr(u), L.ptr(g), L.ptr(b),
            L.ptr(self.X), L.ptr(R), int(e0), int(e1), self.sys._stream()),
            "ldg_operator_pass_range")

    def apply(self, u, tangent, t=0.0, out=None, exchange=True):
        p = self.plan
        u = u.reshape(p.ne_loc, self.n_nodes, self.ncu)
        if not u.is_contiguous():
            u = u.contiguous()
        R = out if out is not None else self.sys._empty((p.ne_loc, self.n_nodes, self.ncu))
        a, b = p.interior
        if not exchange:                       # halos filled by the caller
            self._pass(1, u, tangent, t, R, 0, p.ne_loc)
            return R
        pend = self.start_u_halo(u)
        self._pass(1, u, tangent, t, R, a, b)
        pend.wait()
        self._pass(1, u, tangent, t, R, 0, a)
        self._pass(1, u, tangent, t, R, b, p.ne_loc)
        pend = self.start_x_halo()
        self._pass(2, u, tangent, t, R, a, b)
        pend.wait()
        self._pass(2, u, tangent, t, R, 0, a)
        self._pass(2, u, tangent, t, R, b, p.ne_loc)
        return R

    # -- native halos: the exchange inside the C call (ldg_apply_dist) ---------------------
    def _native_plan(self):
        """ldg_set_halo_plan from the PartitionPlan lists (peers ascending;
        u rows of width ncu, export rows of width nfn * ncu)."""
        import ctypes as C
        from . import _lib as L
        p = self.plan
        peers = sorted(set(p.u_send) | set(p.u_recv) | set(p.x_send) | set(p.x_recv))

        def flat(d):
            rows = [np.asarray(d.get(q, np.zeros(0)), dtype=np.int64) for q in peers]
            off = np.zeros(len(peers) + 1, dtype=np.int64)
            off[1:] = np.cumsum([r.size for r in rows]) if rows else []
            idx = np.concatenate(rows) if rows else np.zeros(0, dtype=np.int64)
            return off, np.ascontiguousarray(idx)
        arrs = [flat(d) for d in (p.u_send, p.u_recv, p.x_send, p.x_recv)]
        self._native_keep = arrs
        ptrs = []
        for off, idx in arrs:
            ptrs += [off.ctypes.data_as(C.c_void_p), idx.ctypes.data_as(C.c_void_p)]
        pr = np.asarray(peers, dtype=np.int32)
        self._native_keep.append(pr)
        a, b = p.interior
        L.check(self.sys.lib.ldg_set_halo_plan(
            self.sys._h, p.ne_loc, int(a), int(b), L.ptr(self.u_ghost), self.ncu,
            self._xper // p.nf, len(peers), pr.ctypes.data_as(C.c_void_p), *ptrs),
            "ldg_set_halo_plan")

    def attach_native_comm(self, group=None):
        """NCCL communicator inside the library (ldg_comm_init): rank 0's
        unique id broadcast over the process group, then the halo plan."""
        import ctypes as C
        import torch.distributed as dist
        from . import _lib as L
        idb = (C.c_uint8 * 128)()
        if self.plan.rank == 0:
            L.check(self.sys.lib.ldg_comm_unique_id(idb), "ldg_comm_unique_id")
        obj = [bytes(idb)]
        dist.broadcast_object_list(obj, src=0, group=group)
        idb = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        L.check(self.sys.lib.ldg_comm_init(self.sys._h, self.plan.nranks, self.plan.rank, idb),
                "ldg_comm_init")
        self._native_plan()
        self.native = True

    def apply_native(self, u, tangent, t=0.0, out=None):
        """The operator with both halo exchanges inside ldg_apply_dist (same
        schedule as :meth:`apply`)."""
        from . import _lib as L
        p = self.plan
        u = u.reshape(p.ne_loc, self.n_nodes, self.ncu)
        if not u.is_contiguous():
            u = u.contiguous()
        R = out if out is not None else self.sys._empty((p.ne_loc, self.n_nodes, self.ncu))
        g = None if tangent else self.sys.boundary_data(t)
        b = None if tangent else self.sys.source_data(t)
        L.check(self.sys.lib.ldg_apply_dist(self.sys._h, int(bool(tangent)), L.ptr(u), L.ptr(g),
                                            L.ptr(b), L.ptr(self.X), L.ptr(R),
                                            self.sys._stream()), "ldg_apply_dist")
        return R

    def complete(self, u, tangent, t=0.0, R=None):
        """Pass 2 over all owned elements (after the caller's export halo)."""
        self._pass(2, u, tangent, t, R, 0, self.plan.ne_loc)
        return R

    native = False          # True once attach_native_comm: halos inside ldg_apply_dist

    def residual_dev(self, u, t=0.0, out=None):
        if self.native:
            return self.apply_native(u, False, t, out)
        return self.apply(u, False, t, out)

    def tangent_dev(self, du, out=None, base=None, t=0.0):
        """Linear fused operator: the tangent reads neither base nor t."""
        if self.native:
            return self.apply_native(du, True, 0.0, out)
        return self.apply(du, True, 0.0, out)


def link_native_local(parts):
    """In-process transport of the native halos (ldg_comm_init_local): the
    partitions' handles act as ranks 0..n-1 of one device; drive each
    partition's apply_native from its own host thread."""
    import ctypes as C
    from . import _lib as L
    hs = (C.c_void_p * len(parts))(*[p.sys._h.value for p in parts])
    L.check(parts[0].sys.lib.ldg_comm_init_local(hs, len(parts)), "ldg_comm_init_local")
    for p in parts:
        p._native_plan()


class LocalDenseTables:
    """DenseTables interface over one partition (simplex elements): rows
    sliced, neighbours renumbered to [owned | ghosts], the element-independent
    operators shared."""

    def __init__(self, tab, plan):
        self._g, self.plan = tab, plan
        for k in ("kind", "nd", "p", "ncu", "nb", "nqf", "nf", "perms", "perm_pts", "dr", "kr",
                  "minv", "lift", "fluxop", "phif", "phio", "au", "aq", "flux_uses_u",
                  "mass_const", "mass_coef", "source_zero", "model", "master", "mesh", "topo",
                  "bc_groups", "face_area_ref", "geom_master"):
            setattr(self, k, getattr(tab, k, None))
        e0, e1 = plan.e0, plan.e1
        self.ne = plan.ne_loc
        self.fnbr, self.finfo, self.ftau = plan.fnbr, plan.finfo, plan.ftau
        self.geo = plan.geo
        self.fnorm, self.fsj = tab.fnorm[e0:e1], tab.fsj[e0:e1]
        self.detj, self.invjt = tab.detj[e0:e1], tab.invjt[e0:e1]
        self.J, self.x0 = tab.J[e0:e1], tab.x0[e0:e1]
        self.elem_vol = tab.elem_vol[e0:e1]
        self.switch, self.fi_h, self.fb_h = tab.switch, tab.fi_h, tab.fb_h
        self.curved = False

    def node_coords(self, elems=None, nodes=None):
        e = np.arange(self.plan.e0, self.plan.e1) if elems is None else \
            np.asarray(elems) + self.plan.e0
        return self._g.node_coords(e, nodes)

    def boundary_values(self, t):
        g = self._g.boundary_values(t)
        return g[self.plan.brows] if g.size else g

    def source_load(self, t):
        b = self._g.source_load(t)
        return None if b is None else b[self.plan.e0:self.plan.e1]


class PartitionedDenseSystem:
    """One rank's share of a simplex (tri / tet) system: owned elements plus
    a ghost layer, the dense mixed and flux passes with whole-row halos of u
    and of the mixed gradient q in between (the flux pass reads the
    neighbours' q).  Neighbour rows >= n_owned come from the halo buffers
    (``ldg_set_ghost_rows_dense``), so the owned vector is used in place."""

    def __init__(self, model, mesh, topology, master, nranks, rank, device=None,
                 exchanger=None, tables=None):
        import torch
        from . import _lib as L
        from .system import LdgSystem
        from .tables import DenseTables
        gtab = tables if tables is not None else DenseTables(model, mesh, topology, master)
        self.plan = PartitionPlan(gtab, nranks, rank)
        self.local = LocalDenseTables(gtab, self.plan)
        self.sys = LdgSystem(model, mesh, topology, master, device=device, tables=self.local)
        self.exchanger = exchanger if exchanger is not None else FaceHaloExchanger(self.plan)
        p = self.plan
        self.n_elements, self.n_nodes, self.ncu, self.nd = p.ne_loc, master.n_nodes, model.ncu, mesh.nd
        self.n_dofs = p.ne_loc * master.n_nodes * model.ncu
        self.kind, self.model, self.device = model.kind, model, self.sys.device
        ng = max(p.n_ghost, 1)
        self.u_ghost = torch.zeros((ng, self.n_nodes, self.ncu), dtype=torch.float64,
                                   device=self.device)
        self.q_ghost = torch.zeros((ng, self.n_nodes, self.ncu, self.nd), dtype=torch.float64,
                                   device=self.device)
        L.check(self.sys.lib.ldg_set_ghost_rows_dense(self.sys._h, p.ne_loc, L.ptr(self.u_ghost),
                                                      L.ptr(self.q_ghost)),
                "ldg_set_ghost_rows_dense")

    def start_u_halo(self, u):
        p = self.plan
        return self.exchanger.start(u.reshape(p.ne_loc, -1), self.u_ghost.view(self.u_ghost.shape[0], -1),
                                    p.row_send, p.row_recv)

    def start_q_halo(self, q):
        p = self.plan
        return self.exchanger.start(q.reshape(p.ne_loc, -1), self.q_ghost.view(self.q_ghost.shape[0], -1),
                                    p.row_send, p.row_recv)

    def apply(self, u, tangent, t=0.0, out=None, exchange=True):
        """R(u) or J du: u halo, mixed pass (owned), q halo, flux pass."""
        p = self.plan
        u = u.reshape(p.ne_loc, self.n_nodes, self.ncu).contiguous()
        if exchange:
            self.start_u_halo(u).wait()
        q = self.sys.mixed_dev(u, t, homogeneous=tangent)
        if exchange:
            self.start_q_halo(q).wait()
        return self.sys.flux_from_mixed_dev(u, q, tangent, t, out=out)

    def residual_dev(self, u, t=0.0, out=None):
        return self.apply(u, False, t, out)

    def tangent_dev(self, du, out=None, base=None, t=0.0):
        return self.apply(du, True, 0.0, out)


class LocalBus:
    """Single-process stand-in for the halo exchange among R partitions
    living on one GPU (partition and halo logic testable without
    8 GPUs): ghost rows (generated path) or ghost face nodes / export slots
    (fused path, the same lists the NCCL exchanger ships) are copied
    device-to-device from the owners."""

    def __init__(self, parts):
        self.parts = parts

    def fill(self, getter):
        for p in self.parts:
            plan = p.plan
            arr = getter(p)
            flat = arr.reshape(arr.shape[0], -1)
            for k, g in enumerate(plan.ghosts.tolist()):
                q = int(plan.owner[g])
                src = getter(self.parts[q])
                flat[plan.ne_loc + k].copy_(src.reshape(src.shape[0], -1)[g - self.parts[q].plan.e0])

    def _lists(self, srcs, dsts, send, recv):
        import torch
        for r, p in enumerate(self.parts):
            for q, rows in getattr(p.plan, recv).items():
                srows = getattr(self.parts[q].plan, send)[r]
                dev = dsts[r].device
                vals = srcs[q].index_select(0, torch.as_tensor(srows, device=dev))
                dsts[r].index_copy_(0, torch.as_tensor(rows, device=dev), vals)

    def apply_all(self, us, tangent, t=0.0):
        """Operator on every partition in lockstep (pass 1 -> exports -> pass 2)."""
        us = [u.reshape(p.plan.ne_loc, p.n_nodes, p.ncu).contiguous()
              for p, u in zip(self.parts, us)]
        self._lists([u.reshape(-1, p.ncu) for p, u in zip(self.parts, us)],
                    [p.u_ghost.view(-1, p.ncu) for p in self.parts], "u_send", "u_recv")
        Rs = [p.apply(u, tangent, t, exchange=False) for p, u in zip(self.parts, us)]
        xs = [p.x_rows() for p in self.parts]
        self._lists(xs, xs, "x_send", "x_recv")
        return [p.complete(u, tangent, t, R) for p, u, R in zip(self.parts, us, Rs)]


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


class PartitionedPackedSystem(PartitionedNlSystem):
    """A partitioned generated-kernel system with packed [u | q | w] states
    (kind W: q is a state; pointwise ODE blocks w): the residual / tangent
    of the u block read the neighbours' u, q and w (face traces, w^ = the
    mean), so those blocks get ghost rows; the gradient equation of kind W
    reads the neighbours' u; the ODE block, the mass and its inverse are
    element- or node-local (disc.py:595-653, 866-948)."""

    @property
    def nw(self):
        return self.model.nw

    @property
    def multi_block(self):
        return self.kind == "W" or self.model.nw > 0

    def block_sizes(self):
        ne, nb = self.plan.ne_loc, self.n_nodes
        sizes = [ne * nb * self.ncu]
        if self.kind == "W":
            sizes.append(ne * nb * self.ncu * self.nd)
        if self.nw > 0:
            sizes.append(ne * nb * self.nw)
        return sizes

    @property
    def n_packed(self):
        return int(sum(self.block_sizes()))

    def unpack(self, Y):
        ne, nb = self.plan.ne_loc, self.n_nodes
        sizes = self.block_sizes()
        parts, o = [], 0
        for k in sizes:
            parts.append(Y[o:o + k])
            o += k
        u = parts[0].reshape(ne, nb, self.ncu)
        q = parts[1].reshape(ne, nb, self.ncu, self.nd) if self.kind == "W" else None
        w = parts[-1].reshape(ne, nb, self.nw) if self.nw > 0 else None
        return u, q, w

    @staticmethod
    def _cat(parts):
        import torch
        return torch.cat([p.reshape(-1) for p in parts if p is not None])

    def _ext(self, a):
        """(owned, ...) -> (owned + ghost, ...) with the ghost rows filled."""
        if a is None:
            return None
        ext = self._new((self.plan.ne_loc + self.plan.n_ghost,) + tuple(a.shape[1:]))
        ext[: self.plan.ne_loc].copy_(a)
        self._exchange(ext)
        return ext

    def residual_packed_dev(self, Y, t=0.0):
        u, q, w = self.unpack(Y)
        ue, we = self._ext(u), self._ext(w)
        if self.kind == "D":
            qe = self.mixed_ext(ue, t)
        else:
            qe = self._ext(q)
        ne = self.plan.ne_loc
        Ru = self.nl.residual(ue, t, q=qe, w=we)[:ne]
        Rq = self.nl.gradient_residual(ue, qe, t) if self.kind == "W" else None
        Rw = self.nl.ode(ue, qe, we, t)[:ne] if self.nw > 0 else None
        return self._cat([Ru, None if Rq is None else Rq[:ne], Rw])

    def tangent_packed_dev(self, V, Y, t=0.0):
        u, q, w = self.unpack(Y)
        du, dq, dw = self.unpack(V)
        ue, we, due, dwe = self._ext(u), self._ext(w), self._ext(du), self._ext(dw)
        if self.kind == "D":
            qe = self.mixed_ext(ue, t)
            dqe = self.mixed_ext(due, t, homogeneous=True)
        else:
            qe, dqe = self._ext(q), self._ext(dq)
        ne = self.plan.ne_loc
        dRu = self.nl.tangent(ue, due, t, q=qe, w=we, dq=dqe, dw=dwe)[:ne]
        dRq = self.nl.gradient_residual(due, dqe, t, tangent=True)[:ne] if self.kind == "W" \
            else None
        dRw = self.nl.ode(ue, qe, we, t, du=due, dq=dqe, dw=dwe)[:ne] if self.nw > 0 else None
        return self._cat([dRu, dRq, dRw])

    def mass_packed_dev(self, V, Y, t=0.0, scale=1.0):
        u, _, _ = self.unpack(Y)
        vu, vq, vw = self.unpack(V)
        Mu = self.nl.mass(vu, u, t, scale)
        Mq = self.nl.mass_q(vq, scale) if self.kind == "W" else None
        Mw = (scale * self.model.ode.alpha) * vw if self.nw > 0 else None
        return self._cat([Mu, Mq, Mw])

    def mass_inv_packed_dev(self, V):
        vu, vq, vw = self.unpack(V)
        return self._cat([self.nl.mass_inv(vu),
                          self.nl.mass_inv_q(vq) if self.kind == "W" else None,
                          vw / self.model.ode.alpha if self.nw > 0 else None])


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


# ---------------------------------------------------------------------------
# distributed steady solve (fused linear path)
# ---------------------------------------------------------------------------


def block_jacobi_partitioned(psys, colors_global):
    """Element block-Jacobi of one rank (solver.py:303-346 on the owned
    blocks): the GLOBAL distance-2 colouring restricted to the owned
    elements, every probe through the partitioned tangent WITH its halos.
    (A rank-local probe is not enough: a ghost neighbour's face export
    depends on the owned element's probe through the shared face's jump, and
    that export is computed on the ghost's owner.)  All ranks run the same
    number of colours and probes, so the halo exchanges pair up."""
    import torch
    from .solver import build_block_jacobi
    p = psys.plan
    colors = np.asarray(colors_global)[p.e0:p.e1]
    ncol = int(np.max(colors_global)) + 1
    x = torch.zeros(psys.n_dofs, dtype=torch.float64, device=psys.device)
    shape = (psys.n_elements, psys.n_nodes, psys.ncu)
    M = build_block_jacobi(lambda xb, v: psys.tangent_dev(v.reshape(shape)).reshape(-1), x,
                           p.ne_loc, psys.n_nodes * psys.ncu, colors, all_colors=ncol)
    torch.cuda.synchronize(psys.device)
    return M


def run_steady_partitioned(psys, precond="block_jacobi", abs_tol=1e-11, rel_tol=3e-8,
                           forcing=1e-8, restart=250, gmres_max_iter=6000, max_iter=20,
                           orth="dcgs2", group=None):
    """driver.run_steady on one rank of an element-partitioned system:
    Newton-GMRES with allreduced Krylov reductions (DistVecOps), rank-local
    block-Jacobi (global colouring), halos every operator application.
    Returns (u owned, stats, timings)."""
    import time
    import torch
    from .driver import DriverError
    from .solver import NewtonOptions, distance2_coloring_topology, newton_solve, vecops
    if psys.kind != "D" or not psys.model.is_steady():
        raise DriverError("partitioned steady solves need a steady kind-D model")
    t0 = time.perf_counter()
    st = psys.sys.interpolate_initial_dev()
    shape = (psys.n_elements, psys.n_nodes, psys.ncu)
    u0 = st.u.reshape(-1)
    ops = DistVecOps(vecops(psys.device), group)
    torch.cuda.synchronize(psys.device)
    t1 = time.perf_counter()
    M = None
    if precond == "block_jacobi":
        tab = psys.local._g
        colors = distance2_coloring_topology(tab.topo, tab.ne)
        M = block_jacobi_partitioned(psys, colors)
    elif precond not in ("identity", None):
        raise DriverError(f"unsupported partitioned preconditioner {precond!r}")
    t2 = time.perf_counter()
    opts = NewtonOptions(abs_tol=abs_tol, rel_tol=rel_tol, max_iter=max_iter, forcing=forcing,
                         gmres_restart=restart, gmres_max_iter=gmres_max_iter,
                         jv_mode="tangent", orth=orth)
    x, stats = newton_solve(lambda v: psys.residual_dev(v.reshape(shape)).reshape(-1), u0, opts,
                            precond=M,
                            tangent_fn=lambda xb, v: psys.tangent_dev(v.reshape(shape)).reshape(-1),
                            ops=ops)
    torch.cuda.synchronize(psys.device)
    t3 = time.perf_counter()
    return x.reshape(shape), stats, {"init_s": t1 - t0, "precond_build_s": t2 - t1,
                                     "solve_s": t3 - t2}
