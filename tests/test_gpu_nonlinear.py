"""Generated-kernel path (nonlinear.py + csrc/ldg_nl.cuh via NVRTC) on the
B200 against reference golden vectors and the oracle.

Bar (BASELINE.json north_star): residual vectors to 1e-12 relative L2 in
fp64.  Cases: kind C Euler / Burgers with the LLF flux (interior, periodic
and Dirichlet ghost states), kind D compressible Navier-Stokes (2D builtin,
3D user model file) with Dirichlet / Neumann / periodic faces, and a
nonlinear diffusion model with state-dependent source and mass, abs / max /
pow / tanh subgradient rules, switch and centered traces."""

import numpy as np
import pytest

from cases import CURVED_CASES, GOLDEN, NL_CASES, b200_setup, build_case, case_state

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def system_for(spec):
    from paper_2205_07824_b200.system import LdgSystem
    return LdgSystem(*build_case(spec, *b200_setup()))


@pytest.mark.parametrize("name", sorted(NL_CASES))
def test_generated_path_vs_reference_golden(name):
    from paper_2205_07824_b200.system import SolverState
    g = np.load(GOLDEN / f"{name}.npz")
    s = system_for(NL_CASES[name])
    assert s.nl is not None, "expected the generated-kernel path"
    assert np.array_equal(s.fi_switch, g["switch"])
    t = float(g["t"])
    st = SolverState(u=g["u"], q=None, w=None, t=t)
    R = s.residual(st)[0]
    J = s.residual_tangent(st, g["du"])[0]
    assert rel(R, g["R"]) < TOL, rel(R, g["R"])
    assert rel(J, g["Jdu"]) < TOL, rel(J, g["Jdu"])
    assert rel(s.mass_apply(st, g["y"])[0], g["M"]) < TOL
    if "Mx" in g:
        assert rel(s.mass_tangent_extra(st, g["y"], g["du"]), g["Mx"]) < TOL
    else:
        assert s.mass_tangent_extra(st, g["y"], g["du"]) is None
    if "q" in g:
        assert rel(s.compute_mixed(g["u"], t), g["q"]) < TOL
        assert rel(s.compute_mixed(g["du"], t, homogeneous=True), g["dq"]) < TOL


@pytest.mark.parametrize("name,counts,p", [
    ("euler2d_quad_periodic_p3", [7, 5], 4),
    ("ns2d_quad_mixedbc_p2", [5, 6], 3),
    ("ns3d_hex_periodic_p2", [3, 3, 2], 3),
    ("euler3d_hex_periodic_p2", [3, 2, 3], 3),
    ("nonlin_diff2d_quad_p2", [6, 5], 5),
])
def test_generated_path_vs_oracle_larger(name, counts, p):
    from oracle import make_oracle
    from paper_2205_07824_b200.system import SolverState
    spec = dict(NL_CASES[name], counts=counts, p=p)
    model, mesh, topo, master = build_case(spec, *b200_setup())
    from paper_2205_07824_b200.system import LdgSystem
    s = LdgSystem(model, mesh, topo, master)
    o = make_oracle(model, mesh, topo, master)
    ne, nb, ncu = s.n_elements, s.n_nodes, s.ncu
    u = case_state(spec, ne, nb, ncu, 5)
    du = np.random.default_rng(6).normal(size=u.shape)
    st = SolverState(u=u, q=None, w=None, t=0.1)
    assert rel(s.residual(st)[0], o.residual(u, 0.1)) < TOL
    assert rel(s.residual_tangent(st, du)[0], o.residual_tangent(u, du, 0.1)) < TOL


def test_tangent_matches_central_difference():
    """disc.py tangent vs central FD of the residual (test_disc.py:320-369
    bar 3e-6) on the 3D Navier-Stokes model.  The reference linearisation
    freezes the wavespeed penalty (disc.py:694-698), so the comparison drops
    the wavespeed to make the tangent the exact derivative."""
    import torch
    from paper_2205_07824_b200.system import LdgSystem, SolverState
    spec = NL_CASES["ns3d_hex_periodic_p2"]
    model, mesh, topo, master = build_case(spec, *b200_setup())
    model.wavespeed = None
    model._plans = {}
    s = LdgSystem(model, mesh, topo, master)
    u = case_state(spec, s.n_elements, s.n_nodes, s.ncu, 3)
    du = np.random.default_rng(4).normal(size=u.shape)
    J = s.residual_tangent(SolverState(u=u, q=None, w=None, t=0.0), du)[0]
    h = 1e-6
    Rp = s.residual(SolverState(u=u + h * du, q=None, w=None, t=0.0))[0]
    Rm = s.residual(SolverState(u=u - h * du, q=None, w=None, t=0.0))[0]
    assert rel((Rp - Rm) / (2 * h), J) < 3e-6
    # device-resident closures give the same numbers
    ud = torch.as_tensor(u, device="cuda")
    Jd = s.tangent_dev(torch.as_tensor(du, device="cuda"), base=ud).cpu().numpy()
    assert rel(Jd, J) < 1e-15


def test_nonfinite_state_raises_kernel_nan():
    from paper_2205_07824_b200.system import KernelNanError, SolverState
    spec = NL_CASES["euler2d_quad_periodic_p3"]
    s = system_for(spec)
    u = case_state(spec, s.n_elements, s.n_nodes, s.ncu, 1)
    u[4, 2, 0] = -1.0            # negative density -> sqrt of a negative pressure ratio
    with pytest.raises(KernelNanError, match="non-finite values"):
        s.residual(SolverState(u=u, q=None, w=None, t=0.0))


def test_generated_kernels_do_not_spill():
    s = system_for(NL_CASES["ns3d_hex_periodic_p2"])
    for k in ("nl_mixed", "nl_residual", "nl_tangent", "nl_mass", "nl_mass_inv"):
        a = s.nl.kernel_attrs(k)
        assert a["regs"] > 0
        print(k, a)


@pytest.mark.parametrize("name", sorted(__import__("cases").MB_CASES))
def test_packed_blocks_vs_reference_golden(name):
    """Kind W (wave: q and w are states; Dirichlet + absorbing faces) and a
    kind D model with a pointwise ODE block: (Ru, Rq, Rw), the tangent
    blocks and (Mu, Mq, Mw) against the reference (disc.py:595-948)."""
    from cases import MB_CASES
    from paper_2205_07824_b200.system import SolverState
    g = np.load(GOLDEN / f"{name}.npz")
    s = system_for(MB_CASES[name])
    assert s.multi_block
    t = float(g["t"])
    get = lambda k: g[k] if k in g else None  # noqa: E731
    st = SolverState(u=g["u"], q=get("q"), w=get("w"), t=t)
    for tag, blocks in (("R", s.residual(st)),
                        ("J", s.residual_tangent(st, g["du"], get("dq"), get("dw"))),
                        ("M", s.mass_apply(st, g["du"], get("dq"), get("dw")))):
        for b, val in zip("uqw", blocks):
            key = f"{tag}{b}"
            if key in g:
                assert val is not None, key
                assert rel(val, g[key]) < TOL, (key, rel(val, g[key]))
            else:
                assert val is None, key


@pytest.mark.parametrize("name,nparts", [("euler2d_quad_periodic_p3", 3),
                                         ("ns2d_quad_mixedbc_p2", 2),
                                         ("ns3d_hex_periodic_p2", 2),
                                         ("nonlin_diff2d_quad_p2", 3)])
def test_partitioned_generated_operator_single_gpu(name, nparts):
    """R element partitions of a generated-kernel model on one GPU (two halo
    steps by device copies: u, then the mixed gradient) assemble to the
    reference operator."""
    import torch
    from paper_2205_07824_b200.nonlinear import NlTables
    from paper_2205_07824_b200.parallel import PartitionedNlSystem, nl_apply_all
    g = np.load(GOLDEN / f"{name}.npz")
    parts_in = build_case(NL_CASES[name], *b200_setup())
    tab = NlTables(*parts_in)
    parts = [PartitionedNlSystem(*parts_in, nranks=nparts, rank=r, tables=tab, exchanger=False)
             for r in range(nparts)]
    t = float(g["t"])
    sl = [slice(p.plan.e0, p.plan.e1) for p in parts]
    us = [torch.as_tensor(g["u"][s], device="cuda") for s in sl]
    dus = [torch.as_tensor(g["du"][s], device="cuda") for s in sl]
    R = np.concatenate([r.cpu().numpy() for r in nl_apply_all(parts, us, False, t=t)])
    J = np.concatenate([r.cpu().numpy() for r in nl_apply_all(parts, dus, True, bases=us, t=t)])
    assert rel(R, g["R"]) < TOL, rel(R, g["R"])
    assert rel(J, g["Jdu"]) < TOL, rel(J, g["Jdu"])


def _nl_rank(rank, world, port, name, out):
    import os
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2205_07824_b200.parallel import PartitionedNlSystem
        g = np.load(GOLDEN / f"{name}.npz")
        parts_in = build_case(NL_CASES[name], *b200_setup())
        s = PartitionedNlSystem(*parts_in, nranks=world, rank=rank)
        sl = slice(s.plan.e0, s.plan.e1)
        t = float(g["t"])
        u = torch.as_tensor(g["u"][sl], device="cuda")
        du = torch.as_tensor(g["du"][sl], device="cuda")
        R = s.residual_dev(u, t).cpu().numpy()
        J = s.tangent_dev(du, base=u, t=t).cpu().numpy()
        np.savez(f"{out}_{rank}.npz", R=R, J=J, e0=s.plan.e0, e1=s.plan.e1)
    finally:
        dist.destroy_process_group()


def test_partitioned_generated_operator_two_ranks_gloo(tmp_path):
    """Two processes sharing the GPU, halos through torch.distributed point to
    point (gloo staging), assemble to the reference operator."""
    import socket
    import torch.multiprocessing as mp
    sck = socket.socket()
    sck.bind(("127.0.0.1", 0))
    port = sck.getsockname()[1]
    sck.close()
    name = "ns3d_hex_periodic_p2"
    out = str(tmp_path / "part")
    mp.start_processes(_nl_rank, args=(2, port, name, out), nprocs=2, start_method="spawn")
    g = np.load(GOLDEN / f"{name}.npz")
    R = np.concatenate([np.load(f"{out}_{r}.npz")["R"] for r in range(2)])
    J = np.concatenate([np.load(f"{out}_{r}.npz")["J"] for r in range(2)])
    assert rel(R, g["R"]) < TOL
    assert rel(J, g["Jdu"]) < TOL


@pytest.mark.parametrize("name", sorted(CURVED_CASES))
def test_curved_elements_vs_reference_golden(name):
    """Non-affine elements (per-point metrics, disc.py:91-180) on the
    generated path vs the unmodified reference on the same mesh: the curved
    O-grid annulus (shallow water, Dirichlet, the reference's acceptance
    criterion 6 on quads) and a periodically warped p_geom = 2 hex box
    (Euler, and Navier-Stokes / Poisson for the quadrature-form mixed
    gradient).  Topology and switch bits bit-exact; the free-stream residual
    vanishes like the reference's (<= 1e-10, criterion 6's bar; the
    reference reaches ~6e-15); R, J du and M y at a perturbed state to 1e-12."""
    from paper_2205_07824_b200.system import LdgSystem, SolverState
    spec = CURVED_CASES[name]
    g = np.load(GOLDEN / spec["mesh_file"])
    model, mesh, topo, master = build_case(spec, *b200_setup())
    s = LdgSystem(model, mesh, topo, master)
    assert s.tab.curved
    assert np.array_equal(np.asarray(topo.elem_l), g["elem_l"])
    assert np.array_equal(s.tab.switch, g["switch"])
    if "u_free" in g:
        Rf = s.residual(SolverState(u=g["u_free"], q=None, w=None, t=0.0))[0]
        assert np.abs(Rf).max() <= 1e-10, np.abs(Rf).max()
    st = SolverState(u=g["u"], q=None, w=None, t=0.0)
    if "q" in g:                  # kind D: the quadrature-form mixed gradient, M_e^-1
        assert rel(s.compute_mixed(g["u"], 0.0), g["q"]) < TOL
        assert rel(s.compute_mixed(g["du"], 0.0, homogeneous=True), g["dq"]) < TOL
    assert rel(s.residual(st)[0], g["R"]) < TOL
    assert rel(s.residual_tangent(st, g["du"])[0], g["Jdu"]) < TOL
    if np.abs(g["M"]).max() > 0:
        assert rel(s.mass_apply(st, g["y"])[0], g["M"]) < TOL


def test_curved_mass_inverse_roundtrip():
    """MassPreconditioner on curved elements: the per-element inverse mass
    (disc.py:107-110) undoes mass_apply."""
    import torch
    from paper_2205_07824_b200.driver import MassPreconditioner
    from paper_2205_07824_b200.system import LdgSystem
    spec = CURVED_CASES["curved_sw_annulus_quad_p3"]
    s = LdgSystem(*build_case(spec, *b200_setup()))
    y = torch.as_tensor(np.random.default_rng(3).normal(size=(s.n_elements, s.n_nodes, s.ncu)),
                        device="cuda")
    My = s.mass_apply_dev(y)
    back = MassPreconditioner(s).apply(My.reshape(-1)).reshape(y.shape)
    assert float(torch.linalg.vector_norm(back - y) / torch.linalg.vector_norm(y)) < 1e-12


def _packed_rank(rank, world, port, name, out):
    import os
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cases import MB_CASES
        from paper_2205_07824_b200.parallel import PartitionedPackedSystem
        g = np.load(GOLDEN / f"{name}.npz")
        s = PartitionedPackedSystem(*build_case(MB_CASES[name], *b200_setup()), nranks=world,
                                    rank=rank)
        sl = slice(s.plan.e0, s.plan.e1)
        t = float(g["t"])

        def packed(pre):
            parts = [torch.as_tensor(g[f"{pre}{b}"][sl], device="cuda").reshape(-1)
                     for b in ("u", "q", "w") if f"{pre}{b}" in g]
            return torch.cat(parts)
        Y = torch.cat([torch.as_tensor(g[k][sl], device="cuda").reshape(-1)
                       for k in ("u", "q", "w") if k in g])
        V = torch.cat([torch.as_tensor(g[k][sl], device="cuda").reshape(-1)
                       for k in ("du", "dq", "dw") if k in g])
        res = {}
        for tag, vec in (("R", s.residual_packed_dev(Y, t)), ("J", s.tangent_packed_dev(V, Y, t)),
                         ("M", s.mass_packed_dev(V, Y, t))):
            u, q, w = s.unpack(vec)
            for b, val in zip("uqw", (u, q, w)):
                if val is not None:
                    res[f"{tag}{b}"] = val.cpu().numpy()
        np.savez(f"{out}_{rank}.npz", e0=s.plan.e0, **res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["wave2d_quad_absorbing_p3", "wave3d_hex_periodic_p2",
                                  "reactode2d_quad_p2"])
def test_partitioned_packed_blocks_two_ranks_gloo(tmp_path, name):
    """Kind W (q a state) and ODE-block systems partitioned over two ranks
    sharing the GPU: ghost rows of u, q and w, the gradient equation and the
    ODE block owned-only; the assembled (R, J, M) blocks equal the reference
    goldens (disc.py:595-948)."""
    import socket
    import torch.multiprocessing as mp
    sck = socket.socket()
    sck.bind(("127.0.0.1", 0))
    port = sck.getsockname()[1]
    sck.close()
    out = str(tmp_path / "packed")
    mp.start_processes(_packed_rank, args=(2, port, name, out), nprocs=2, start_method="spawn")
    g = np.load(GOLDEN / f"{name}.npz")
    parts = [np.load(f"{out}_{r}.npz") for r in range(2)]
    for key in ("Ru", "Rq", "Rw", "Ju", "Jq", "Jw", "Mu", "Mq", "Mw"):
        if key in g:
            val = np.concatenate([p[key] for p in parts])
            assert rel(val, g[key]) < TOL, (key, rel(val, g[key]))
