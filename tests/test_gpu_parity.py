"""B200 kernels vs the reference (golden vectors) and vs the oracle.

Bar (BASELINE.json north_star): residual vectors agree to 1e-12 relative
L2 in fp64; connectivity and switch bits bit-exact."""

import numpy as np
import pytest

from cases import CASES, GOLDEN, b200_setup, build_case

pytestmark = pytest.mark.gpu
TENSOR = sorted(CASES)            # every case: tensor (quad/hex) and dense (tri/tet) paths
TOL = 1e-12


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def system_for(name):
    from paper_2205_07824_b200.system import LdgSystem
    return LdgSystem(*build_case(CASES[name], *b200_setup()))


@pytest.mark.parametrize("name", TENSOR)
def test_residual_tangent_mixed_vs_reference_golden(name):
    from paper_2205_07824_b200.system import SolverState
    g = np.load(GOLDEN / f"{name}.npz")
    s = system_for(name)
    assert np.array_equal(s.fi_switch, g["switch"])
    st = SolverState(u=g["u"], q=None, w=None, t=0.0)
    R, _, _ = s.residual(st)
    J, _, _ = s.residual_tangent(st, g["du"])
    assert isinstance(R, np.ndarray) and R.shape == g["R"].shape
    assert rel(R, g["R"]) < TOL
    assert rel(J, g["Jdu"]) < TOL
    assert rel(s.compute_mixed(g["u"], 0.0), g["q"]) < TOL
    assert rel(s.compute_mixed(g["du"], 0.0, homogeneous=True), g["dq"]) < TOL


@pytest.mark.parametrize("kind,counts,p", [("hex", [7, 6, 5], 3), ("hex", [5, 4, 6], 1),
                                          ("hex", [4, 4, 3], 4), ("hex", [3, 3, 4], 5),
                                          ("quad", [13, 9], 3), ("quad", [6, 7], 6),
                                          ("tri", [7, 6], 3), ("tri", [5, 5], 4),
                                          ("tet", [4, 3, 3], 3), ("tet", [3, 3, 3], 1)])
def test_vs_oracle_poisson_larger(kind, counts, p):
    from oracle import make_oracle
    from paper_2205_07824_b200 import meshgen, model, refelem
    from paper_2205_07824_b200.system import LdgSystem, SolverState
    nd = len(counts)
    m = model.load_model(str(GOLDEN / f"poisson{nd}d.model"))
    mesh = meshgen.generate_structured([(0.0, 1.0)] * nd, counts, kind)
    topo = meshgen.build_face_topology(mesh)
    master = refelem.build_master(kind, p)
    s = LdgSystem(m, mesh, topo, master)
    o = make_oracle(m, mesh, topo, master)
    rng = np.random.default_rng(7)
    u = rng.normal(size=(s.n_elements, s.n_nodes, 1))
    du = rng.normal(size=u.shape)
    st = SolverState(u=u, q=None, w=None, t=0.0)
    assert rel(s.residual(st)[0], o.residual(u)) < TOL
    assert rel(s.residual_tangent(st, du)[0], o.residual_tangent(u, du)) < TOL


def test_convdiff_periodic_p1_to_p5_vs_oracle():
    from cases import BOX_PERIODIC
    from oracle import make_oracle
    from paper_2205_07824_b200 import meshgen, model, refelem
    from paper_2205_07824_b200.system import LdgSystem, SolverState
    m = model.builtin_model("convection_diffusion", nd=3, mu=[1.0, 1.0, 1.0, 1.0])
    m.bcs = {}
    for p, n in ((1, 6), (2, 5), (3, 4), (4, 3), (5, 3)):
        mesh = meshgen.generate_structured([(0.0, 1.0)] * 3, [n] * 3, "hex")
        topo = meshgen.build_face_topology(mesh, BOX_PERIODIC[3])
        master = refelem.build_master("hex", p)
        s = LdgSystem(m, mesh, topo, master)
        o = make_oracle(m, mesh, topo, master)
        rng = np.random.default_rng(p)
        u = rng.normal(size=(s.n_elements, s.n_nodes, 1))
        st = SolverState(u=u, q=None, w=None, t=0.0)
        assert rel(s.residual_tangent(st, u)[0], o.residual_tangent(u, u)) < TOL, p


@pytest.mark.parametrize("p", [1, 2, 3])
@pytest.mark.parametrize("model_name", ["poisson", "convection_diffusion"])
def test_sheared_hex_vs_oracle(model_name, p):
    """Affinely sheared hexes: the element coefficient blocks C = detJ J^-T A J^-1
    are full 3x3 (the plane kernels' general-C branch; axis-aligned boxes take
    the diagonal branch); p = 1, 2: plane_kernel_g, p = 3: plane_kernel."""
    from oracle import make_oracle
    from paper_2205_07824_b200 import meshgen, model, refelem
    from paper_2205_07824_b200.system import LdgSystem, SolverState
    if model_name == "poisson":
        m = model.load_model(str(GOLDEN / "poisson3d.model"))
    else:
        m = model.builtin_model("convection_diffusion", nd=3, mu=[0.6, -0.3, 0.4, 0.7])
        m.bcs = {t: model.BoundaryCondition(type="dirichlet", data=["x1*x3 - 0.2*x2"])
                 for t in range(1, 7)}
    mesh = meshgen.generate_structured([(0.0, 1.0)] * 3, [4, 3, 5], "hex")
    A = np.array([[1.0, 0.3, 0.1], [0.0, 1.0, 0.2], [0.0, 0.0, 0.9]])
    mesh.vertices = mesh.vertices @ A.T
    mesh.ho_nodes = mesh.ho_nodes @ A.T
    topo = meshgen.build_face_topology(mesh)
    master = refelem.build_master("hex", p)
    s = LdgSystem(m, mesh, topo, master)
    o = make_oracle(m, mesh, topo, master)
    rng = np.random.default_rng(11)
    u = rng.normal(size=(s.n_elements, s.n_nodes, 1))
    du = rng.normal(size=u.shape)
    st = SolverState(u=u, q=None, w=None, t=0.0)
    assert rel(s.residual(st)[0], o.residual(u)) < TOL
    assert rel(s.residual_tangent(st, du)[0], o.residual_tangent(u, du)) < TOL


def test_device_path_is_deterministic_and_linear_at_scale():
    """Size-independent properties at a config-3-like size: bitwise
    run-to-run reproducibility and linearity of the tangent."""
    import torch
    from paper_2205_07824_b200 import meshgen, model, refelem
    from paper_2205_07824_b200.system import LdgSystem
    m = model.load_model(str(GOLDEN / "poisson3d.model"))
    mesh = meshgen.generate_structured([(0.0, 1.0)] * 3, [24] * 3, "hex")
    s = LdgSystem(m, mesh, meshgen.build_face_topology(mesh), refelem.build_master("hex", 3))
    g = torch.Generator(device="cuda").manual_seed(3)
    shape = (s.n_elements, s.n_nodes, 1)
    a = torch.randn(shape, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(shape, dtype=torch.float64, device="cuda", generator=g)
    Ja, Ja2 = s.tangent_dev(a), s.tangent_dev(a)
    assert torch.equal(Ja, Ja2)
    Jb = s.tangent_dev(b)
    Jab = s.tangent_dev(1.5 * a - 0.25 * b)
    err = torch.linalg.norm(Jab - (1.5 * Ja - 0.25 * Jb)) / torch.linalg.norm(Jab)
    assert float(err) < 1e-13


@pytest.mark.parametrize("name", ["poisson3d_hex_p2", "poisson3d_hex_p3"])
def test_nan_reported_with_element(name):
    """hex p=2: pencil kernel; hex p=3: plane kernel + warp completion
    kernel (integer exponent test, one atomic per thread)."""
    from paper_2205_07824_b200.system import KernelNanError, SolverState
    s = system_for(name)
    u = np.zeros((s.n_elements, s.n_nodes, 1))
    u[5, 3, 0] = np.nan
    with pytest.raises(KernelNanError, match="non-finite values"):
        s.residual(SolverState(u=u, q=None, w=None, t=0.0))
    u[5, 3, 0] = np.inf
    with pytest.raises(KernelNanError, match="non-finite values"):
        s.residual_tangent(SolverState(u=u, q=None, w=None, t=0.0), u)


@pytest.mark.parametrize("name,nparts", [("poisson3d_hex_p3", 3), ("convdiff3d_hex_periodic_p2", 4),
                                         ("poisson2d_quad_p3", 2), ("poisson3d_hex_centered_p2", 3)])
def test_partitioned_native_operator_single_gpu(name, nparts):
    """R partitions on one GPU (native fused passes, ghosts by device copies)
    assemble to the reference operator."""
    import torch
    from paper_2205_07824_b200.parallel import LocalBus, PartitionedLdgSystem
    from paper_2205_07824_b200.tables import TensorTables
    g = np.load(GOLDEN / f"{name}.npz")
    parts_in = build_case(CASES[name], *b200_setup())
    tab = TensorTables(*parts_in)
    parts = [PartitionedLdgSystem(*parts_in, nranks=nparts, rank=r, tables=tab, exchanger=False)
             for r in range(nparts)]
    bus = LocalBus(parts)
    for key, tangent, want in (("u", False, "R"), ("du", True, "Jdu")):
        us = [torch.as_tensor(g[key][p.plan.e0:p.plan.e1], device="cuda") for p in parts]
        Rs = bus.apply_all(us, tangent)
        R = np.concatenate([r.cpu().numpy() for r in Rs])
        assert rel(R, g[want]) < TOL, (key, rel(R, g[want]))


@pytest.mark.parametrize("name,nparts", [("poisson3d_tet_p2", 3), ("poisson2d_tri_p2", 2),
                                         ("poisson3d_tet_p2", 2)])
def test_partitioned_dense_operator_single_gpu(name, nparts):
    """R partitions of a simplex system on one GPU (dense mixed / flux
    passes, ghost u and q rows by device copies of the same row lists the
    NCCL exchanger ships) assemble to the reference operator."""
    import torch
    from paper_2205_07824_b200.parallel import LocalBus, PartitionedDenseSystem
    from paper_2205_07824_b200.tables import DenseTables
    g = np.load(GOLDEN / f"{name}.npz")
    parts_in = build_case(CASES[name], *b200_setup())
    tab = DenseTables(*parts_in)
    parts = [PartitionedDenseSystem(*parts_in, nranks=nparts, rank=r, tables=tab, exchanger=False)
             for r in range(nparts)]
    bus = LocalBus(parts)
    for key, tangent, want in (("u", False, "R"), ("du", True, "Jdu")):
        us = [torch.as_tensor(g[key][p.plan.e0:p.plan.e1], device="cuda").contiguous()
              for p in parts]
        bus._lists([u.reshape(u.shape[0], -1) for u in us],
                   [p.u_ghost.view(p.u_ghost.shape[0], -1) for p in parts], "row_send", "row_recv")
        qs = [p.sys.mixed_dev(u, 0.0, homogeneous=tangent) for p, u in zip(parts, us)]
        bus._lists([q.reshape(q.shape[0], -1) for q in qs],
                   [p.q_ghost.view(p.q_ghost.shape[0], -1) for p in parts], "row_send", "row_recv")
        Rs = [p.sys.flux_from_mixed_dev(u, q, tangent, 0.0) for p, u, q in zip(parts, us, qs)]
        R = np.concatenate([r.cpu().numpy() for r in Rs])
        assert rel(R, g[want]) < TOL, (key, rel(R, g[want]))


def test_host_pipeline_matches_device_and_never_aliases():
    """Pinned-CPU torch inputs run the chunk-pipelined ldg_apply_host (H2D,
    passes and D2H overlapped): bitwise equal to the device path, and a result
    the caller still holds is never reused for a later call."""
    import torch
    from paper_2205_07824_b200 import meshgen, model, refelem
    from paper_2205_07824_b200.system import LdgSystem, SolverState
    m = model.load_model(str(GOLDEN / "poisson3d.model"))
    mesh = meshgen.generate_structured([(0.0, 1.0)] * 3, [20, 18, 16], "hex")
    s = LdgSystem(m, mesh, meshgen.build_face_topology(mesh), refelem.build_master("hex", 3))
    assert len(s._pipe_plan()[1]) > 1
    shape = (s.n_elements, s.n_nodes, 1)
    a = torch.randn(shape, dtype=torch.float64).pin_memory()
    b = torch.randn(shape, dtype=torch.float64).pin_memory()
    st = SolverState(u=a, q=None, w=None, t=0.0)
    Ja = s.residual_tangent(st, a)[0]
    Ja_copy = Ja.clone()
    Jb = s.residual_tangent(st, b)[0]
    Jc = s.residual_tangent(st, a)[0]
    assert Ja.data_ptr() != Jb.data_ptr() and Jc.data_ptr() not in (Ja.data_ptr(), Jb.data_ptr())
    assert torch.equal(Ja, Ja_copy) and torch.equal(Jc, Ja)
    assert torch.equal(Jb, s.tangent_dev(b.cuda()).cpu())
    Ra = s.residual(st)[0]
    assert torch.equal(Ra, s.residual_dev(a.cuda()).cpu())


@pytest.mark.parametrize("name", ["poisson3d_hex_p3", "poisson2d_quad_p3", "poisson2d_tri_p2",
                                  "poisson3d_tet_p2", "convdiff2d_quad_dirichlet_p2"])
def test_device_source_matches_host_restatement(name):
    """source_dev.DeviceSource (plan on the device) == tables.source_load
    (numpy restatement of disc.py:621-629)."""
    from paper_2205_07824_b200.source_dev import DeviceSource
    s = system_for(name)
    if getattr(s.tab, "source_zero", False):
        pytest.skip("model without a source")
    dev = DeviceSource(s.tab, s.device).load(0.3).cpu().numpy()
    host = s.tab.source_load(0.3)
    assert rel(dev, host) < 1e-13


@pytest.mark.parametrize("shear", [False, True])
def test_hex_p3_vs_oracle_at_scale(shear):
    """The config-3 kernels past one persistent sweep: 30x28x26 hexes = 2,730
    eight-element groups against the plane kernel's grid of 1,184 warps (and
    the completion kernel's), so every warp runs the double-buffered loop at
    least twice (buffer 1, prefetch of group g + stride).  Axis-aligned: the
    DIAG branch; sheared: the general-C branch.  Oracle R and J du at 1e-12."""
    from oracle import make_oracle
    from paper_2205_07824_b200 import meshgen, model, refelem
    from paper_2205_07824_b200.system import LdgSystem, SolverState
    m = model.load_model(str(GOLDEN / "poisson3d.model"))
    mesh = meshgen.generate_structured([(0.0, 1.0)] * 3, [30, 28, 26], "hex")
    if shear:
        A = np.array([[1.0, 0.3, 0.1], [0.0, 1.0, 0.2], [0.0, 0.0, 0.9]])
        mesh.vertices = mesh.vertices @ A.T
        mesh.ho_nodes = mesh.ho_nodes @ A.T
    topo = meshgen.build_face_topology(mesh)
    master = refelem.build_master("hex", 3)
    s = LdgSystem(m, mesh, topo, master)
    assert s.n_elements // 8 > 2 * 1184
    o = make_oracle(m, mesh, topo, master)
    rng = np.random.default_rng(17)
    u = rng.normal(size=(s.n_elements, s.n_nodes, 1))
    du = rng.normal(size=u.shape)
    st = SolverState(u=u, q=None, w=None, t=0.0)
    assert rel(s.residual(st)[0], o.residual(u)) < TOL
    assert rel(s.residual_tangent(st, du)[0], o.residual_tangent(u, du)) < TOL


@pytest.mark.parametrize("p,counts,sweep", [(2, [32, 32, 30], 148 * 5 * 2 * 10),
                                            (1, [40, 40, 36], 148 * 3 * 4 * 16)])
def test_hex_p1_p2_vs_oracle_at_scale(p, counts, sweep):
    """plane_kernel_g (hex p = 1, 2, config 5) past one persistent sweep:
    more than twice the elements one sweep of its grid covers (MINB blocks
    per SM x warps per block x 32 / N1 elements per warp), so every warp runs
    the double-buffered loop at least twice; also the last partial group
    (p = 2: 10 elements per warp).  Oracle R and J du at 1e-12."""
    from oracle import make_oracle
    from paper_2205_07824_b200 import meshgen, model, refelem
    from paper_2205_07824_b200.system import LdgSystem, SolverState
    m = model.builtin_model("convection_diffusion", nd=3, mu=[0.6, -0.3, 0.4, 0.7])
    m.bcs = {t: model.BoundaryCondition(type="dirichlet", data=["x1*x3 - 0.2*x2"])
             for t in range(1, 7)}
    mesh = meshgen.generate_structured([(0.0, 1.0)] * 3, counts, "hex")
    topo = meshgen.build_face_topology(mesh)
    master = refelem.build_master("hex", p)
    s = LdgSystem(m, mesh, topo, master)
    assert s.n_elements > 2 * sweep
    o = make_oracle(m, mesh, topo, master)
    rng = np.random.default_rng(19)
    u = rng.normal(size=(s.n_elements, s.n_nodes, 1))
    du = rng.normal(size=u.shape)
    st = SolverState(u=u, q=None, w=None, t=0.0)
    assert rel(s.residual(st)[0], o.residual(u)) < TOL
    assert rel(s.residual_tangent(st, du)[0], o.residual_tangent(u, du)) < TOL


@pytest.mark.parametrize("option,value,p", [("pass1_variant", 1, 3), ("c_diag", 0, 3), ("p2_mode", 1, 3),
                                            ("p2_mode", 2, 3), ("p2_mode", 3, 3),
                                            ("pass1_variant", 1, 2), ("c_diag", 0, 2),
                                            ("pass1_variant", 1, 1), ("c_diag", 0, 1),
                                            ("p2_mode", 1, 1)])
def test_kernel_variants_equal_default(option, value, p):
    """Every kernel variant ldg_set_option selects (the pencil pass 1, the
    general flux-coefficient branch on an axis-aligned mesh, pass 2 without
    PDL / block-wise / one-shot) gives the default operator to 1e-13 on a
    hex p=3 mesh past one persistent sweep."""
    import torch
    from paper_2205_07824_b200 import meshgen, model, refelem
    from paper_2205_07824_b200.system import LdgSystem
    m = model.load_model(str(GOLDEN / "poisson3d.model"))
    counts = {3: [24, 22, 20], 2: [32, 32, 30], 1: [40, 40, 36]}[p]
    mesh = meshgen.generate_structured([(0.0, 1.0)] * 3, counts, "hex")
    s = LdgSystem(m, mesh, meshgen.build_face_topology(mesh), refelem.build_master("hex", p))
    du = torch.as_tensor(np.random.default_rng(5).normal(size=(s.n_elements, s.n_nodes, 1)),
                         device="cuda")
    u = torch.as_tensor(np.random.default_rng(6).normal(size=du.shape), device="cuda")
    ref_j, ref_r = s.tangent_dev(du).clone(), s.residual_dev(u).clone()
    assert s.lib.ldg_set_option(s._h, option.encode(), value) == 0
    assert rel(s.tangent_dev(du).cpu().numpy(), ref_j.cpu().numpy()) < 1e-13
    assert rel(s.residual_dev(u).cpu().numpy(), ref_r.cpu().numpy()) < 1e-13
    assert s.lib.ldg_set_option(s._h, b"no_such_option", 1) != 0


def test_fused_equals_unfused_at_config3_size():
    """Config 3 (hex p=3, n=54, 10,077,696 DOFs) on the device: the fused
    two-pass matvec (q never leaves the SM) against the unfused reference
    structure (compute_mixed -> flux from q, disc.py:601-653), both for the
    tangent and for the residual with source and Dirichlet data."""
    import torch
    from paper_2205_07824_b200 import meshgen, model, refelem
    from paper_2205_07824_b200.system import LdgSystem
    m = model.load_model(str(GOLDEN / "poisson3d.model"))
    mesh = meshgen.generate_structured([(0.0, 1.0)] * 3, [54] * 3, "hex")
    s = LdgSystem(m, mesh, meshgen.build_face_topology(mesh), refelem.build_master("hex", 3))
    assert s.n_dofs == 10_077_696
    g = torch.Generator(device="cuda").manual_seed(0)
    du = torch.randn((s.n_elements, s.n_nodes, 1), dtype=torch.float64, device="cuda",
                     generator=g)
    J = s.tangent_dev(du)
    dq = s.mixed_dev(du, 0.0, homogeneous=True)
    Ju = s.flux_from_mixed_dev(du, dq, True)
    assert float(torch.linalg.norm(J - Ju) / torch.linalg.norm(Ju)) < TOL
    R = s.residual_dev(du, 0.0)
    q = s.mixed_dev(du, 0.0)
    Ru = s.flux_from_mixed_dev(du, q, False, 0.0)
    assert float(torch.linalg.norm(R - Ru) / torch.linalg.norm(Ru)) < TOL


def _threaded(fns):
    """Run callables concurrently, one host thread (and one CUDA stream)
    each, like ranks; returns their results in order."""
    import threading
    import torch
    out, err = [None] * len(fns), []

    def run(i):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                out[i] = fns[i]()
                torch.cuda.current_stream().synchronize()
        except Exception as e:          # surfaced below
            err.append(e)
    ts = [threading.Thread(target=run, args=(i,)) for i in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert not err, err
    assert all(not t.is_alive() for t in ts), "a rank hung"
    return out


@pytest.mark.parametrize("name,nparts", [("poisson3d_hex_p3", 3), ("convdiff3d_hex_periodic_p2", 4),
                                         ("poisson2d_quad_p3", 2)])
def test_native_halos_in_process_match_reference(name, nparts):
    """ldg_apply_dist (both halo exchanges inside the C call, the in-process
    transport of ldg_comm_init_local standing in for NCCL on a one-GPU pool):
    partitions driven from concurrent host threads assemble to the
    reference operator, over repeated calls (the mailbox rounds)."""
    import torch
    from paper_2205_07824_b200.parallel import PartitionedLdgSystem, link_native_local
    from paper_2205_07824_b200.tables import TensorTables
    g = np.load(GOLDEN / f"{name}.npz")
    parts_in = build_case(CASES[name], *b200_setup())
    tab = TensorTables(*parts_in)
    parts = [PartitionedLdgSystem(*parts_in, nranks=nparts, rank=r, tables=tab, exchanger=False)
             for r in range(nparts)]
    link_native_local(parts)
    for _ in range(2):
        for key, tangent, want in (("u", False, "R"), ("du", True, "Jdu")):
            us = [torch.as_tensor(g[key][p.plan.e0:p.plan.e1], device="cuda").contiguous()
                  for p in parts]
            Rs = _threaded([lambda p=p, u=u: p.apply_native(u, tangent) for p, u in zip(parts, us)])
            R = np.concatenate([r.cpu().numpy() for r in Rs])
            assert rel(R, g[want]) < TOL, (key, rel(R, g[want]))


@pytest.mark.parametrize("nparts", [2, 3])
def test_native_halos_in_process_match_global_at_scale(nparts):
    """hex p=3 n=8 (interior ranges overlap the halos): ldg_apply_dist on
    2 / 3 in-process ranks vs the single-GPU operator, bit for bit up to the
    summation order (1e-13)."""
    import torch
    from paper_2205_07824_b200.parallel import PartitionedLdgSystem, link_native_local
    from paper_2205_07824_b200.system import LdgSystem
    from paper_2205_07824_b200.tables import TensorTables
    spec = dict(model=("file", "poisson3d.model"), kind="hex", counts=[8, 8, 8], p=3)
    parts_in = build_case(spec, *b200_setup())
    tab = TensorTables(*parts_in)
    s = LdgSystem(*parts_in, tables=tab)
    parts = [PartitionedLdgSystem(*parts_in, nranks=nparts, rank=r, tables=tab, exchanger=False)
             for r in range(nparts)]
    assert any(p.plan.interior[1] > p.plan.interior[0] for p in parts)
    link_native_local(parts)
    gen = torch.Generator(device="cuda").manual_seed(5)
    u = torch.randn((s.n_elements, s.n_nodes, 1), dtype=torch.float64, device="cuda", generator=gen)
    want = s.tangent_dev(u).cpu().numpy()
    want_r = s.residual_dev(u).cpu().numpy()
    for _ in range(3):
        Rs = _threaded([lambda p=p: p.apply_native(u[p.plan.e0:p.plan.e1], True) for p in parts])
        assert rel(np.concatenate([r.cpu().numpy() for r in Rs]), want) < 1e-13
        Rs = _threaded([lambda p=p: p.apply_native(u[p.plan.e0:p.plan.e1], False) for p in parts])
        assert rel(np.concatenate([r.cpu().numpy() for r in Rs]), want_r) < 1e-13


def test_native_comm_nccl_single_rank():
    """The NCCL transport end to end on a one-rank communicator: libnccl
    dlopen'ed, unique id broadcast over torch.distributed, ncclCommInitRank,
    the halo plan (no peers) and ldg_apply_dist equal the single-GPU
    operator."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_2205_07824_b200.parallel import PartitionedLdgSystem
    from paper_2205_07824_b200.system import LdgSystem
    from paper_2205_07824_b200.tables import TensorTables
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", world_size=1, rank=0)
    try:
        spec = dict(model=("file", "poisson3d.model"), kind="hex", counts=[4, 4, 4], p=3)
        parts_in = build_case(spec, *b200_setup())
        tab = TensorTables(*parts_in)
        s = LdgSystem(*parts_in, tables=tab)
        p = PartitionedLdgSystem(*parts_in, nranks=1, rank=0, tables=tab, exchanger=False)
        p.attach_native_comm()
        u = torch.randn((s.n_elements, s.n_nodes, 1), dtype=torch.float64, device="cuda")
        assert rel(p.apply_native(u, True).cpu().numpy(), s.tangent_dev(u).cpu().numpy()) < 1e-13
        assert rel(p.apply_native(u, False).cpu().numpy(), s.residual_dev(u).cpu().numpy()) < 1e-13
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("model_name,shear", [("poisson", False), ("poisson", True),
                                              ("convection_diffusion", False)])
def test_one_launch_operator_bitwise_equal_two_launch(model_name, shear):
    """The one-launch operator (plane_kernel<.., FUSED>, ldg_set_option "fused"):
    pass 2 of each 8-element group runs in the same persistent launch once the
    pass-1 windows it reads are published.  Same arithmetic in the same order
    as plane_kernel + complete_warp4_kernel, so R and J du are BITWISE equal to
    the two-launch operator, over repeated launches (the claim / window
    counters reset themselves at the end of each launch), at a size past one
    persistent sweep (2,730 groups vs 1,184 warps); DIAG, general-C and
    convective (Cu) branches."""
    import torch
    from paper_2205_07824_b200 import meshgen, model, refelem
    from paper_2205_07824_b200.system import LdgSystem
    if model_name == "poisson":
        m = model.load_model(str(GOLDEN / "poisson3d.model"))
    else:
        m = model.builtin_model("convection_diffusion", nd=3, mu=[0.6, -0.3, 0.4, 0.7])
        m.bcs = {t: model.BoundaryCondition(type="dirichlet", data=["x1*x3 - 0.2*x2"])
                 for t in range(1, 7)}
    mesh = meshgen.generate_structured([(0.0, 1.0)] * 3, [30, 28, 26], "hex")
    if shear:
        A = np.array([[1.0, 0.3, 0.1], [0.0, 1.0, 0.2], [0.0, 0.0, 0.9]])
        mesh.vertices = mesh.vertices @ A.T
        mesh.ho_nodes = mesh.ho_nodes @ A.T
    s = LdgSystem(m, mesh, meshgen.build_face_topology(mesh), refelem.build_master("hex", 3))
    rng = np.random.default_rng(23)
    du = torch.as_tensor(rng.normal(size=(s.n_elements, s.n_nodes, 1)), device="cuda")
    u = torch.as_tensor(rng.normal(size=du.shape), device="cuda")
    out = {}
    for fused in (0, 1):
        assert s.lib.ldg_set_option(s._h, b"fused", fused) == 0
        out[fused] = [(s.tangent_dev(du).clone(), s.residual_dev(u).clone()) for _ in range(3)]
    for k in range(3):
        assert torch.equal(out[1][k][0], out[0][0][0])
        assert torch.equal(out[1][k][1], out[0][0][1])
