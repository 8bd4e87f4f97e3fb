"""Multi-process (world_size 2, gloo, CPU) tests of the element-partitioned
layer: partition tables, halo exchanges and allreduced Krylov reductions,
with the fused operator's arithmetic emulated in numpy (no GPU).  The
assembled partitioned results must equal the global operator (reference
golden vectors) and the distributed Newton-GMRES must reproduce the
single-process iteration counts and solution."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class CpuOps:
    """VecOps semantics on CPU tensors (the CUDA kernels' reference)."""

    def dot(self, x, y, out):
        out.fill_(float(x @ y))

    def nrm2(self, x, out):
        out.fill_(float(torch.linalg.vector_norm(x)))

    def norm(self, x):
        return float(torch.linalg.vector_norm(x))

    def axpy(self, a, x, y, a_dev=None, sign=1.0):
        y.add_(x, alpha=float(a) if a_dev is None else sign * float(a_dev))

    def div(self, x, den, out):
        torch.div(x, den, out=out)

    def div_guarded(self, x, den, thr, out):
        if float(den) > thr:
            torch.div(x, den, out=out)

    def mgs_step(self, vi, h_in, w, vnext, h_out):
        if vi is not None:
            w.sub_(h_in * vi)
        if vnext is not None:
            h_out.fill_(float(vnext @ w))

    def cgs_dots(self, V, k, w, h):
        h[:k] = V[:k] @ w

    def cgs_update(self, V, k, h, w, nrm):
        w.sub_(h[:k] @ V[:k])
        if nrm is not None:
            nrm.fill_(float(torch.linalg.vector_norm(w)))

    def combine(self, Z, k, y, x):
        x.add_(y[:k] @ Z[:k])

    def dcgs_dots(self, V, k, x, y, hx, hy):
        hx[:k] = V[:k] @ x
        hy[:k] = V[:k] @ y

    def dcgs_update(self, V, m, s, t, v, w, out, inv_alpha, gamma, nrm):
        vf = (v - s[:m] @ V[:m]) * inv_alpha
        v.copy_(vf)
        out.copy_((w - t[:m] @ V[:m] - gamma * vf) * inv_alpha)
        if nrm is not None:
            nrm.fill_(float(torch.linalg.vector_norm(out)))


def _worker(rank, world, port, name, q, orth):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(__file__))
        import tensor_emulation as emu
        from cases import CASES, GOLDEN, b200_setup, build_case
        from paper_2205_07824_b200.parallel import (DistVecOps, FaceHaloExchanger, LocalTables,
                                                    PartitionPlan)
        from paper_2205_07824_b200.tables import TensorTables
        g = np.load(GOLDEN / f"{name}.npz")
        tab = TensorTables(*build_case(CASES[name], *b200_setup()))
        plan = PartitionPlan(tab, world, rank)
        loc = LocalTables(tab, plan)
        halo = FaceHaloExchanger(plan)
        ne_ext = plan.ne_loc + plan.n_ghost
        nb, ncu = g["u"].shape[1:]
        gp = loc.boundary_projection(0.0)
        bs = loc.source_load(0.0)

        def apply(uvec, tangent):
            # face-node halos: only the ghost face nodes the cut faces read
            # are filled (the rest of u_ext's ghost rows stays zero) and only
            # the export slot facing this rank; the result must still be exact
            u_ext = torch.zeros((ne_ext, nb, ncu), dtype=torch.float64)
            u_ext[:plan.ne_loc] = uvec.reshape(plan.ne_loc, nb, ncu)
            halo.start(u_ext[:plan.ne_loc].reshape(-1, ncu), u_ext[plan.ne_loc:].reshape(-1, ncu),
                       plan.u_send, plan.u_recv).wait()
            R, X = emu.pass1(loc, u_ext.numpy(), tangent, None if tangent else gp,
                             None if tangent else bs)
            X_ext = torch.zeros((ne_ext,) + X.shape[1:], dtype=torch.float64)
            X_ext[:plan.ne_loc] = torch.as_tensor(X)
            xr = X_ext.reshape(ne_ext * X.shape[1], -1)
            halo.start(xr, xr, plan.x_send, plan.x_recv).wait()
            return torch.as_tensor(emu.pass2(loc, X_ext.numpy(), R)).reshape(-1)

        e0, e1 = plan.e0, plan.e1
        u = torch.as_tensor(g["u"][e0:e1]).reshape(-1)
        du = torch.as_tensor(g["du"][e0:e1]).reshape(-1)
        R = apply(u, False).reshape(-1, nb, ncu).numpy()
        J = apply(du, True).reshape(-1, nb, ncu).numpy()
        err = max(np.abs(R - g["R"][e0:e1]).max() / np.abs(g["R"]).max(),
                  np.abs(J - g["Jdu"][e0:e1]).max() / np.abs(g["Jdu"]).max())
        # distributed Newton-GMRES on the partitioned operator
        from paper_2205_07824_b200.solver import NewtonOptions, newton_solve
        ops = DistVecOps(CpuOps())
        opts = NewtonOptions(abs_tol=1e-13, rel_tol=1e-11, forcing=1e-12, gmres_restart=400,
                             gmres_max_iter=2000, jv_mode="tangent", orth=orth)
        x, st = newton_solve(lambda v: apply(v, False), torch.zeros(plan.ne_loc * nb * ncu,
                                                                    dtype=torch.float64),
                             opts, tangent_fn=lambda x_, v: apply(v, True), ops=ops)
        q.put((rank, float(err), st.newton_iters, st.total_gmres_iters, e0, e1,
               x.numpy().copy(), plan.n_ghost, sorted(plan.u_send), sorted(plan.u_recv)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,orth", [("poisson3d_hex_p3", "cgs2"), ("convdiff3d_hex_periodic_p2", "cgs2"),
                                       ("poisson2d_quad_p3", "cgs2"), ("poisson3d_hex_centered_p2", "cgs2"),
                                       ("poisson3d_hex_p3", "dcgs2"), ("convdiff3d_hex_periodic_p2", "dcgs2")])
def test_partitioned_operator_and_solve_gloo(name, orth):
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    import tensor_emulation as emu
    from cases import CASES, b200_setup, build_case
    from paper_2205_07824_b200.solver import NewtonOptions, newton_solve
    from paper_2205_07824_b200.tables import TensorTables
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q, orth)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    for r in res:
        assert r[1] < 1e-13, r[:2]
        assert r[7] > 0 and r[8] and r[9]          # real ghosts and halo lists
    # single-process solve with the same emulated operator and reductions
    tab = TensorTables(*build_case(CASES[name], *b200_setup()))
    gp, bs = tab.boundary_projection(0.0), tab.source_load(0.0)
    shape = (tab.ne, tab.master.n_nodes, tab.ncu)

    def apply(v, tangent):
        u = v.reshape(shape).numpy()
        return torch.as_tensor(emu.fused(tab, u, tangent, None if tangent else gp,
                                         None if tangent else bs)).reshape(-1)

    opts = NewtonOptions(abs_tol=1e-13, rel_tol=1e-11, forcing=1e-12, gmres_restart=400,
                         gmres_max_iter=2000, jv_mode="tangent", orth=orth)
    x, st = newton_solve(lambda v: apply(v, False), torch.zeros(int(np.prod(shape)),
                                                                 dtype=torch.float64),
                         opts, tangent_fn=lambda x_, v: apply(v, True), ops=CpuOps())
    xd = np.concatenate([r[6] for r in res])
    assert all(r[2] == st.newton_iters for r in res)
    assert all(abs(r[3] - st.total_gmres_iters) <= 1 for r in res)
    rel = np.linalg.norm(xd - x.numpy()) / max(np.linalg.norm(x.numpy()), 1e-30)
    print("solution rel diff", rel, st.total_gmres_iters)
    assert rel <= 1e-10


def _dense_worker(rank, world, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(__file__))
        import dense_emulation as emu
        from cases import CASES, GOLDEN, b200_setup, build_case
        from paper_2205_07824_b200.parallel import (FaceHaloExchanger, LocalDenseTables,
                                                    PartitionPlan)
        from paper_2205_07824_b200.tables import DenseTables
        g = np.load(GOLDEN / f"{name}.npz")
        tab = DenseTables(*build_case(CASES[name], *b200_setup()))
        plan = PartitionPlan(tab, world, rank)
        loc = LocalDenseTables(tab, plan)
        halo = FaceHaloExchanger(plan)
        ne_ext = plan.ne_loc + plan.n_ghost
        nb, ncu = g["u"].shape[1:]
        gv = loc.boundary_values(0.0)
        bs = loc.source_load(0.0)
        e0, e1 = plan.e0, plan.e1
        out = {}
        for key, tangent, want in (("u", False, "R"), ("du", True, "Jdu")):
            u_ext = torch.zeros((ne_ext, nb, ncu), dtype=torch.float64)
            u_ext[:plan.ne_loc] = torch.as_tensor(g[key][e0:e1])
            halo.start(u_ext[:plan.ne_loc].reshape(plan.ne_loc, -1),
                       u_ext[plan.ne_loc:].reshape(plan.n_ghost, -1),
                       plan.row_send, plan.row_recv).wait()
            qo = emu.mixed(loc, u_ext.numpy(), None if tangent else gv)
            q_ext = torch.zeros((ne_ext,) + qo.shape[1:], dtype=torch.float64)
            q_ext[:plan.ne_loc] = torch.as_tensor(qo[:plan.ne_loc])
            halo.start(q_ext[:plan.ne_loc].reshape(plan.ne_loc, -1),
                       q_ext[plan.ne_loc:].reshape(plan.n_ghost, -1),
                       plan.row_send, plan.row_recv).wait()
            R = emu.flux(loc, u_ext.numpy(), q_ext.numpy(), tangent, None if tangent else gv,
                         None if tangent else bs)
            out[want] = float(np.abs(R[:plan.ne_loc] - g[want][e0:e1]).max() /
                              np.abs(g[want]).max())
        q.put((rank, out, plan.n_ghost))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["poisson3d_tet_p2", "poisson2d_tri_p2"])
def test_partitioned_dense_operator_gloo(name):
    """Simplex partitions on two processes (gloo): whole-row halos of u and of
    the mixed gradient between the emulated dense passes assemble to the
    reference goldens."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dense_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, errs, ng in res:
        assert ng > 0
        assert errs["R"] < 1e-13 and errs["Jdu"] < 1e-13, (rank, errs)
