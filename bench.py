"""Benchmark: LDG tangent matvec GDOF/s (3D Poisson, hex p=3, ~10M DOFs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A "step" is one Jacobian-vector product J(u) du of the config-3 system
(BASELINE.json configs[2]: 3D Poisson on a structured hex box mesh, p=3,
n=54 -> 10,077,696 DOFs) -- the matvec GMRES applies every iteration.

* ``value``: device-resident throughput (inputs already in HBM), CUDA events
  on the launching stream, max over ranks.  Inputs+outputs (du 81 MB, dq
  242 MB, dR 81 MB) exceed the 126 MB L2, so no flush is needed.
* ``e2e``: the same metric through the public drop-in call
  ``LdgSystem.residual_tangent(state, du)`` with du in pinned host memory and
  the result returned in host memory, copies inside the timed region.
* ``roofline``: the dominant kernel (the flux pass) against measured HBM
  bandwidth with its algorithmic bytes; ``matvec_roofline``: the whole
  matvec at SURVEY 8(d)'s 72 B/DOF.
* ``cpu_baseline``: the oracle (restatement of the reference numpy path) on
  a bounded sample, rank 0 only.
* ``--impl reference``: that reference CPU implementation timed on this
  host, same metric and unit.

Multi-GPU (torchrun, N>1): weak scaling on an N-slab box ((54 N) x 54 x 54
hexes); each rank owns one 10M-DOF x-slab, exchanges ghost-element halos
over NCCL twice per matvec (parallel.PartitionedLdgSystem).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

N_ELEM = 54          # 54^3 hexes x 64 nodes = 10,077,696 DOFs
P = 3
CPU_SAMPLE_N = 10    # 10^3 hexes x 64 nodes = 64,000 DOFs
MODEL = ROOT / "tests" / "golden" / "poisson3d.model"
METRIC = "DG matvec GDOF/s (3D, p=3)"
BYTES_FLUX = 40      # flux pass: du 8 + dq 24 read, dR 8 written (per DOF)
BYTES_MIXED = 32     # mixed pass: du 8 read, dq 24 written
BYTES_MATVEC = 72    # 8 (3 + 2 nd)


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def build_problem(n, p=P, nx_mult=1):
    """Config-3 problem; with nx_mult = N the box is N unit cubes long in x
    (N x-slabs of n^3 elements: weak scaling, one slab per rank)."""
    from paper_2205_07824_b200 import meshgen, model, refelem
    m = model.load_model(str(MODEL))
    mesh = meshgen.generate_structured([(0.0, float(nx_mult)), (0.0, 1.0), (0.0, 1.0)],
                                       [n * nx_mult, n, n], "hex")
    topo = meshgen.build_face_topology(mesh)
    master = refelem.build_master("hex", p)
    return m, mesh, topo, master


def cpu_oracle_times(n, reps):
    """Oracle residual_tangent on n^3 hexes: per-call seconds, DOFs."""
    from oracle import make_oracle
    m, mesh, topo, master = build_problem(n)
    o = make_oracle(m, mesh, topo, master)
    ne, nb = mesh.connectivity.shape[0], master.n_nodes
    u = np.random.default_rng(1).normal(size=(ne, nb, 1))
    du = np.random.default_rng(0).normal(size=(ne, nb, 1))
    o.residual_tangent(u, du)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        o.residual_tangent(u, du)
        ts.append(time.perf_counter() - t0)
    return ts, ne * nb


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.p, self.out = index, None, ""

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p is None:
            return
        self.p.terminate()
        try:
            self.out, _ = self.p.communicate(timeout=5)
        except Exception:
            self.p.kill()

    def summary(self):
        rows = [[x.strip() for x in r.split(",")] for r in self.out.strip().splitlines()
                if r.count(",") >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4)
                          if r[4 + k].lower() in ("active", "1")})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


def run_solve(system, orth="dcgs2"):
    """Newton-GMRES time to solution on the bench system with the
    reference acceptance flags (test_acceptance.py:69-81), block-Jacobi."""
    import torch
    from paper_2205_07824_b200.driver import run_steady
    torch.cuda.synchronize()
    # hand the matvec / e2e phases' cached blocks back to the driver first,
    # so the first solve allocates its 20 GB Krylov workspace like a solve in
    # a fresh process would (outside the timed region)
    torch.cuda.empty_cache()
    st, stats, tm = run_steady(system, precond="block_jacobi", orth=orth)
    torch.cuda.synchronize()
    # the same solve again: Krylov workspace (20 GB at restart 250) and the
    # caching allocator warm, as for every solve after the first
    _, _, tm2 = run_steady(system, precond="block_jacobi", orth=orth)
    torch.cuda.synchronize()
    xq = system.disc.xq
    w = system.disc.wdetj
    uq = np.einsum("qa,ea->eq", system.master.phi, st.u.reshape(system.n_elements, -1).cpu().numpy())
    ex = np.sin(np.pi * xq[..., 0]) * np.sin(np.pi * xq[..., 1]) * np.sin(np.pi * xq[..., 2])
    err = float(np.sqrt(np.sum(w * (uq - ex) ** 2) / np.sum(w * ex ** 2)))
    return {"orth": orth, "precond_build_s": tm["precond_build_s"], "solve_s": tm["solve_s"],
            "time_to_solution_s": tm["precond_build_s"] + tm["solve_s"],
            "warm": {"precond_build_s": tm2["precond_build_s"], "solve_s": tm2["solve_s"],
                     "time_to_solution_s": tm2["precond_build_s"] + tm2["solve_s"]},
            "newton_iters": stats.newton_iters, "gmres_iters": stats.total_gmres_iters,
            "final_residual": stats.final_residual, "error_u": err,
            "bj_blocks": tm.get("bj_blocks"), "bj_inverses": tm.get("bj_inverses")}


def run_strong(args, world, dev, steps=10):
    """Strong scaling beside the weak-scaling headline: the fixed config-3
    box (n^3 hexes in total, 10.08M DOFs at n = 54) split into `world`
    x-slabs, the partitioned tangent matvec timed like the headline (CUDA
    events on the stream, L2 flushed, max over ranks).  GDOF/s of the whole
    box; the driver computes efficiency from per-N values itself."""
    import torch
    import torch.distributed as dist
    from paper_2205_07824_b200.parallel import PartitionedLdgSystem
    m, mesh, topo, master = build_problem(args.n, nx_mult=1)
    ps = PartitionedLdgSystem(m, mesh, topo, master, world, int(os.environ.get("RANK", 0)),
                              device=dev)
    g = torch.Generator(device=dev).manual_seed(7)
    du = torch.randn((ps.n_elements, ps.n_nodes, 1), dtype=torch.float64, device=dev, generator=g)
    dR = torch.empty_like(du)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    for _ in range(3):
        ps.tangent_dev(du, out=dR)
    stream = torch.cuda.current_stream()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(steps)]
    torch.cuda.synchronize()
    dist.barrier()
    for k in range(steps):
        flush.fill_(float(k))
        ev[k][0].record(stream)
        ps.tangent_dev(du, out=dR)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    t = torch.tensor([ms], dtype=torch.float64,
                     device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    total = mesh.connectivity.shape[0] * master.n_nodes
    return {"workload": f"config 3 box n={args.n} (fixed, {total} DOFs) split over {world} ranks",
            "dofs": total, "ms_per_step": ms, "gdofs": total / (ms * 1e-3) / 1e9}


def run_solve_partitioned(s, world):
    """Newton-GMRES time to solution on the N-slab box (each rank one slab;
    allreduced DCGS2, rank-local block-Jacobi, face-node halos), the max over
    ranks of the device-synchronised wall time."""
    import torch
    import torch.distributed as dist
    from paper_2205_07824_b200.parallel import run_steady_partitioned
    u, stats, tm = run_steady_partitioned(s, orth="dcgs2")
    t = torch.tensor([tm["precond_build_s"], tm["solve_s"]], dtype=torch.float64,
                     device=s.device if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    b, sv = (float(x) for x in t.tolist())
    return {"metric": "Newton-GMRES time to solution (s), N-slab config-3 box, block-Jacobi, "
                      "acceptance flags", "dofs": world * s.n_dofs,
            "gpu": {"orth": "dcgs2", "precond_build_s": b, "solve_s": sv,
                    "time_to_solution_s": b + sv, "newton_iters": stats.newton_iters,
                    "gmres_iters": stats.total_gmres_iters,
                    "final_residual": stats.final_residual}}


def cpu_solve(n):
    """Oracle (reference numpy path) steady solve on n^3 hexes, same flags."""
    from oracle import make_oracle
    from oracle.solver_oracle import (block_jacobi_blocks, block_jacobi_factor,
                                      distance2_coloring, element_neighbors, newton_solve)
    m, mesh, topo, master = build_problem(n)
    o = make_oracle(m, mesh, topo, master)
    ne, nb = mesh.connectivity.shape[0], master.n_nodes
    tan = lambda x, v: o.residual_tangent(x.reshape(ne, nb, 1), v.reshape(ne, nb, 1)).ravel()  # noqa: E731
    t0 = time.perf_counter()
    colors = distance2_coloring(element_neighbors(topo, ne))
    M = block_jacobi_factor(block_jacobi_blocks(tan, np.zeros(ne * nb), ne, nb, colors))
    t1 = time.perf_counter()
    x, st = newton_solve(lambda x: o.residual(x.reshape(ne, nb, 1)).ravel(), tan, np.zeros(ne * nb),
                         abs_tol=1e-11, rel_tol=3e-8, forcing=1e-8, restart=250,
                         gmres_max_iter=6000, precond=M)
    t2 = time.perf_counter()
    return {"dofs": ne * nb, "precond_build_s": t1 - t0, "solve_s": t2 - t1,
            "time_to_solution_s": t2 - t0, "newton_iters": st["newton_iters"],
            "gmres_iters": int(sum(st["gmres_iters"])), "cores": 1}


def load_traffic():
    """DRAM bytes per launch of the two fused kernels from the committed ncu
    --set full capture (profiles/traffic.json, written by
    scripts/ncu_traffic.py from the same bench command): dram__bytes_read.sum +
    dram__bytes_write.sum.  Absent file -> null."""
    try:
        return json.loads((ROOT / "profiles" / "traffic.json").read_text())
    except Exception:
        return {}


def fp64_line(p1_ms):
    """FP64 peak measured with a DFMA microbenchmark
    (ldg_probe_fp64) and the pass-1 kernel's FP64 rate from its exact FP64
    operation count (ncu smsp__sass_thread_inst_executed_op_{dfma,dmul,dadd}
    of the same bench command, profiles/fp64_counts.json; an FMA counts 2)."""
    import ctypes
    from paper_2205_07824_b200._lib import load, check
    tf, ms = ctypes.c_double(), ctypes.c_double()
    check(load().ldg_probe_fp64(20000, ctypes.byref(tf), ctypes.byref(ms), None), "fp64 probe")
    out = {"peak_tflops": tf.value, "peak_source": "ldg_probe_fp64 (8 DFMA chains/thread)"}
    try:
        cnt = json.loads((ROOT / "profiles" / "fp64_counts.json").read_text())
        fl = cnt["pass1_flops"]
        out.update({"pass1_flops_per_launch": fl, "pass1_tflops": fl / (p1_ms * 1e-3) / 1e12,
                    "pass1_frac": fl / (p1_ms * 1e-3) / 1e12 / tf.value,
                    "count_source": cnt.get("source")})
    except Exception:
        pass
    return out


def tet_line(hbm, n=44, reps=10):
    """SURVEY 8(d) config-3 tet variant: 3D Poisson on the Kuhn-tet box n=44,
    p=3 (10,222,080 DOFs), tangent J du on the dense simplex kernels
    (csrc/ldg_dense.cu), L2 flushed between reps."""
    import torch
    from paper_2205_07824_b200 import meshgen, model, refelem
    from paper_2205_07824_b200.system import LdgSystem
    t0 = time.perf_counter()
    m = model.load_model(str(ROOT / "tests" / "golden" / "poisson3d.model"))
    mesh = meshgen.generate_structured([(0.0, 1.0)] * 3, [n] * 3, "tet")
    s = LdgSystem(m, mesh, meshgen.build_face_topology(mesh), refelem.build_master("tet", 3))
    setup = time.perf_counter() - t0
    g = torch.Generator(device="cuda").manual_seed(0)
    du = torch.randn((s.n_elements, s.n_nodes, 1), dtype=torch.float64, device="cuda", generator=g)
    out = torch.empty_like(du)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for _ in range(3):
        s.tangent_dev(du, out=out)
    st = torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        s.tangent_dev(du, out=out)
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    nd = s.n_dofs
    return {"workload": f"config 3 tet variant: Kuhn tets n={n}, p=3, tangent J du", "dofs": nd,
            "ms": ms, "gdofs": nd / (ms * 1e-3) / 1e9,
            "matvec_frac_72B": nd * 72 / (ms * 1e-3) / 1e9 / hbm, "setup_s": round(setup, 1)}


def nonlinear_lines(hbm, cpu=True):
    """Configs 4 and 2 on the generated-kernel path (scripts/nl_bench.py):
    3D compressible Navier-Stokes hex p=3 n=32 (10.5M DOFs) and 2D Euler quad
    p=4 n=256 (6.6M DOFs) residual / tangent GDOF/s with the SURVEY 8(d)
    byte counts (104 / 24 B/DOF)."""
    sys.path.insert(0, str(ROOT / "scripts"))
    import nl_bench
    from cases import TRANSIENT_CASES
    out = {}
    ns = dict(TRANSIENT_CASES["ns3d_tgv_hex_p2_dirk11"], counts=[32] * 3, p=3,
              state=([1.0, 0.2, -0.1, 0.15, 25.0], 0.05))
    eu = dict(TRANSIENT_CASES["euler2d_vortex_quad_p3_dirk22"], counts=[256] * 2, p=4,
              state=([1.0, 0.2, -0.1, 2.5], 0.05))
    small = {"config4_ns3d_hex_p3_n32": dict(ns, counts=[3] * 3),
             "config2_euler2d_quad_p4_n256": dict(eu, counts=[6] * 2)}
    for name, spec in (("config4_ns3d_hex_p3_n32", ns), ("config2_euler2d_quad_p4_n256", eu)):
        _, r = nl_bench.run(name, spec, 10, hbm)
        out[name] = {k: r[k] for k in ("dofs", "tangent_gdofs", "residual_gdofs", "tangent_ms",
                                       "residual_ms", "tangent_bytes_per_dof",
                                       "tangent_frac_hbm", "tangent_uncached_gdofs",
                                       "base_cache_ms")}
        if cpu:
            c = nl_bench.cpu_oracle_tangent(small[name])
            out[name]["cpu_baseline"] = dict(c, sample=f"{c['dofs']}-DOF mesh of the same "
                                                      "model / p, oracle tangent")
    # implicit steps (time to solution per step; config 2 is
    # quad p=4 n=64 with DIRK(1,1) = BDF1 and the mass preconditioner; config 4
    # hex p=3 n=16 -- its reference transient block-Jacobi does not converge
    # (DESIGN.md), so the mass preconditioner)
    eu64 = dict(eu, counts=[64] * 2, stages=1, order=1)
    ns16 = dict(ns, counts=[16] * 3, stages=1, order=1)
    out["config2_step_euler_vortex_p4_n64_bdf1"] = nl_bench.run_transient(eu64, 3, 0.01)
    # (dt 0.05 / 0.01 stall Newton within 20 iterations with the frozen-penalty
    # linearisation -- as the reference itself does at n=3, measured -- so
    # config 4 steps at dt = 0.002)
    out["config4_step_ns3d_tgv_p3_n16_bdf1"] = nl_bench.run_transient(ns16, 2, 0.002)
    return out


REF_SRC = ROOT / "baseline" / "_ref"      # the unmodified reference, pip --target install


def _ref_worker(n, steps, warmup, barrier, q):
    """One host process: the UNMODIFIED reference (ldgkit from baseline/_ref)
    LdgSystem.residual_tangent on its own n^3 hex p=3 Poisson box (the
    reference's numpy path, disc.py:591-593).  Steps are synchronised across
    the workers by `barrier`; returns per-step seconds."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    sys.path.insert(0, str(REF_SRC))
    from ldgkit import master as r_master, mesh as r_mesh, model as r_model
    from ldgkit.disc import LdgSystem as RefSystem, SolverState as RefState
    m = r_model.load_model(str(MODEL))
    mesh = r_mesh.generate_structured([(0.0, 1.0)] * 3, [n] * 3, "hex")
    s = RefSystem(m, mesh, r_mesh.build_face_topology(mesh), r_master.build_master("hex", P))
    ne, nb = s.n_elements, s.n_nodes
    u = np.random.default_rng(1).normal(size=(ne, nb, 1))
    du = np.random.default_rng(0).normal(size=(ne, nb, 1))
    st = RefState(u=u, q=None, w=None, t=0.0)
    for _ in range(warmup):
        s.residual_tangent(st, du)
    ts = []
    for _ in range(steps):
        barrier.wait()
        t0 = time.perf_counter()
        s.residual_tangent(st, du)
        ts.append(time.perf_counter() - t0)
    q.put((ne * nb, ts))


def reference_times(n, steps, warmup, procs):
    """The reference's CPU path on `procs` host processes at once (each an
    independent n^3 sample; the reference itself is single-threaded numpy):
    per-step max over processes, total DOFs.  Uses ldgkit from baseline/_ref
    when installed ("reference"), else the oracle port ("port", 1 process)."""
    if not (REF_SRC / "ldgkit").is_dir():
        ts, nd = cpu_oracle_times(n, steps)
        return ts, nd, 1, "port"
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    barrier, q = ctx.Barrier(procs), ctx.Queue()
    ps = [ctx.Process(target=_ref_worker, args=(n, steps, warmup, barrier, q)) for _ in range(procs)]
    for p in ps:
        p.start()
    res = [q.get() for _ in ps]
    for p in ps:
        p.join()
    ts = np.max(np.array([r[1] for r in res]), axis=0)
    return list(ts), sum(r[0] for r in res), procs, "reference"


def ref_procs():
    """All host cores the reference arm may use (bounded: each process holds
    a ~1 GB reference Discretization of the sample)."""
    try:
        c = len(os.sched_getaffinity(0))
    except Exception:
        c = os.cpu_count() or 1
    return max(1, min(c, 64))


def run_reference(args, rank):
    """The reference's own CPU implementation of the path (ldgkit's
    LdgSystem.residual_tangent from baseline/_ref, unmodified), on all the
    host cores: one reference process per core, each on a bounded
    n=CPU_SAMPLE_N sample of config 3, steps synchronised, per-step time the
    max over processes."""
    if rank != 0:
        return
    procs = ref_procs()
    ts, ndof, cores, kind = reference_times(CPU_SAMPLE_N, max(args.steps, 1), args.warmup, procs)
    med = float(np.median(ts))
    v = ndof / med / 1e9
    sample = (f"{cores} processes x {ndof // cores}-DOF hex p=3 Poisson boxes (n={CPU_SAMPLE_N}, "
              f"config 3's model/order) of "
              + ("ldgkit.disc.LdgSystem.residual_tangent (unmodified, baseline/_ref)"
                 if kind == "reference" else "the oracle port (baseline/_ref absent)")
              + f"; median over {len(ts)} synchronised steps of the max over processes")
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": "GDOF/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": med * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config 3 (3D Poisson hex p=3) tangent matvec J(u)du; "
                               f"bounded samples, {ndof} DOFs per step over {cores} cores",
                   "full_size_extrapolation_s": 10077696 / (v * 1e9)},
        "cpu_baseline": {"value": v, "unit": "GDOF/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": v, "unit": "GDOF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def config5_lines(hbm):
    """BASELINE config 5: 3D convection-diffusion tangent matvec, fully
    periodic unit cube, hex p = 1..5 at ~10M DOFs each (scripts/
    sweep_config5.py: CUDA events on the launching stream, L2 flushed
    between reps, median of 10)."""
    import gc
    import torch
    sys.path.insert(0, str(Path(__file__).resolve().parent / "scripts"))
    import sweep_config5
    rows = []
    for p in (1, 2, 3, 4, 5):
        rows.append(sweep_config5.run_p(p, 10, hbm))
        gc.collect()
        torch.cuda.empty_cache()
    return {"metric": "config 5: 3D conv-diff periodic tangent matvec GDOF/s, p = 1..5",
            "unit": "GDOF/s", "rows": rows}


def run_b200(args, rank, world):
    import torch
    import torch.distributed as dist
    from paper_2205_07824_b200 import _lib as L
    from paper_2205_07824_b200.system import LdgSystem, SolverState
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    m, mesh, topo, master = build_problem(args.n, nx_mult=world)
    t0 = time.time()
    if world == 1:
        s = LdgSystem(m, mesh, topo, master)
        core = s
    else:
        # element-partitioned: this rank owns one x-slab, NCCL halos
        from paper_2205_07824_b200.parallel import PartitionedLdgSystem
        s = PartitionedLdgSystem(m, mesh, topo, master, world, rank, device=dev)
        core = s.sys
        if dist.get_backend() == "nccl":
            # halos inside the C call (ldg_apply_dist over the library's own
            # NCCL communicator); torch.distributed halos otherwise
            try:
                s.attach_native_comm()
            except Exception as e:            # NCCL unavailable: keep the torch halos
                print(f"native halos unavailable ({e}); torch.distributed halos", file=sys.stderr)
    setup_s = time.time() - t0
    ne, nb, ndof = s.n_elements, s.n_nodes, s.n_dofs
    gen = torch.Generator(device=dev).manual_seed(rank)
    du = torch.randn((ne, nb, 1), dtype=torch.float64, device=dev, generator=gen)
    dR = torch.empty_like(du)
    X = core.scratch() if world == 1 else s.X
    u_in = du                          # partitioned: ghost rows come from s.u_ghost
    dq = torch.empty((ne, nb, 1, 3), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    lib, h = core.lib, core._h
    if args.fused is not None:
        L.check(lib.ldg_set_option(h, b"fused", int(args.fused)), "fused option")

    def step():
        if world == 1:
            s.tangent_dev(du, out=dR, scratch=X)
        else:
            s.tangent_dev(du, out=dR)

    def launch_pass(k):
        L.check(lib.ldg_operator_pass(h, k, 1, L.ptr(u_in), None, None, L.ptr(X), L.ptr(dR),
                                      L.stream_ptr()), "operator pass")

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)   # 256 MB > L2
    st_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    with ClockSampler(dev.index) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        start.record(stream)
        for k in range(args.steps):
            flush.fill_(float(k))                 # evict L2 between timed steps
            st_ev[k][0].record(stream)
            step()
            st_ev[k][1].record(stream)
        end.record(stream)
        torch.cuda.synchronize()
        # per-kernel split, same stream, events between the two launches
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)]
              for _ in range(args.steps)]
        for k in range(args.steps):
            ev[k][0].record(stream)
            launch_pass(1)
            ev[k][1].record(stream)
            launch_pass(2)
            ev[k][2].record(stream)
        torch.cuda.synchronize()
        # the unfused reference structure (mixed -> flux), same inputs
        ev2 = [[torch.cuda.Event(enable_timing=True) for _ in range(3)]
               for _ in range(args.steps)]
        for k in range(args.steps):
            ev2[k][0].record(stream)
            if world == 1:
                core.mixed_dev(du, homogeneous=True, out=dq)
            ev2[k][1].record(stream)
            if world == 1:
                core.flux_from_mixed_dev(du, dq, True, out=dR)
            ev2[k][2].record(stream)
        torch.cuda.synchronize()
    p1_ms = [e[0].elapsed_time(e[1]) for e in ev]
    p2_ms = [e[1].elapsed_time(e[2]) for e in ev]
    unf_ms = [e[0].elapsed_time(e[2]) for e in ev2]
    unf_mixed = [e[0].elapsed_time(e[1]) for e in ev2]
    t_ms = float(np.sum([e[0].elapsed_time(e[1]) for e in st_ev])) / args.steps
    tmax = torch.tensor([t_ms], dtype=torch.float64,
                        device=dev if dist.is_initialized() and dist.get_backend() == "nccl" else "cpu")
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    t_ms = float(tmax.item())
    traffic = load_traffic()
    p1_name = ("plane_kernel<tangent> (pass 1, z-plane mapping, persistent)"
               if (core.tab.n1 == 4 and core.tab.nd == 3 and core.ncu == 1)
               else "fused_kernel<tangent> (pass 1, pencil mapping)")
    # algorithmic bytes of the fused passes from the face tables
    tab = core.tab
    info = tab.finfo
    interior = (info & 3) == 0
    right = (info & 4) > 0
    sw = (info & 8) > 0
    gcen = m.numflux.grad_trace == "centered"
    exports = int(np.sum(interior & (gcen | (sw == right))))       # faces written in pass 1
    completes = int(np.sum(interior & (gcen | (sw != right))))     # faces read in pass 2
    nfn = tab.nfn
    bytes_p1 = 8 * ndof + 8 * ndof + 8 * exports * nfn
    bytes_p2 = 16 * ndof + 8 * completes * nfn

    # e2e through the public drop-in call with host buffers: numpy in -> numpy
    # out (the reference's calling convention, disc.py:588-593; pageable input
    # staged by the library's host threads) and, beside it, pinned torch CPU
    # tensors
    du_np = du.cpu().numpy()
    du_host = du.cpu().pin_memory()

    def e2e_time(x_host):
        if world == 1:
            st = SolverState(u=x_host, q=None, w=None, t=0.0)

            def e2e_step():
                return s.residual_tangent(st, x_host)[0]
        else:
            out_host = torch.empty(du_host.shape, dtype=torch.float64, pin_memory=True)

            def e2e_step():
                d = torch.as_tensor(x_host).to(dev, non_blocking=True)
                r = s.tangent_dev(d)
                out_host.copy_(r, non_blocking=True)
                torch.cuda.current_stream().synchronize()
                return out_host
        for _ in range(max(args.warmup, 3)):     # same pattern as the timed loop (the caller
            out = e2e_step()                      # holds the previous result)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0 = time.perf_counter()
        ea.record(stream)
        for _ in range(args.steps):
            out = e2e_step()
        eb.record(stream)
        torch.cuda.synchronize()
        ms = ea.elapsed_time(eb) / args.steps
        wall = (time.perf_counter() - e0) / args.steps * 1e3
        assert not (isinstance(out, torch.Tensor) and out.is_cuda)
        emax = torch.tensor([ms], dtype=torch.float64,
                            device=dev if dist.is_initialized() and dist.get_backend() == "nccl"
                            else "cpu")
        if world > 1:
            dist.all_reduce(emax, op=dist.ReduceOp.MAX)
        return float(emax.item()), wall
    e2e_ms, wall_e2e = e2e_time(du_np)
    e2e_pin_ms, wall_pin = e2e_time(du_host)

    solve_line = None
    if world > 1 and not args.no_solve:
        solve_line = run_solve_partitioned(s, world)
    strong_line = run_strong(args, world, dev) if world > 1 else None
    if rank != 0:
        return
    pk = peaks()
    hbm = float(pk.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in pk else "fallback 6.65 TB/s"
    p1 = float(np.median(p1_ms))
    p2 = float(np.median(p2_ms))
    gdofs = world * ndof / (t_ms * 1e-3) / 1e9
    ach_p1 = bytes_p1 / (p1 * 1e-3) / 1e9
    ach_p2 = bytes_p2 / (p2 * 1e-3) / 1e9
    ach_mv = BYTES_MATVEC * ndof / (t_ms * 1e-3) / 1e9
    ach_fused = (bytes_p1 + bytes_p2) / (t_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": gdofs, "unit": "GDOF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded normal du)",
        "config": {"workload": "config 3: 3D Poisson (tests/golden/poisson3d.model) on "
                               f"structured hex box n={args.n}, p=3, tangent J(u)du",
                   "dofs_per_gpu": ndof, "elements_per_gpu": ne,
                   "l2": "L2 flushed (256 MB write) between timed steps; per-step CUDA events",
                   "parallelism": (f"element-partitioned x{world} (x-slabs, "
                                   + ("NCCL halos inside ldg_apply_dist)" if getattr(s, "native", False)
                                      else "torch.distributed halos)")
                                   if world > 1 else "single GPU"),
                   "setup_s": round(setup_s, 2)},
        "e2e": {"value": world * ndof / (e2e_ms * 1e-3) / 1e9, "unit": "GDOF/s",
                "h2d_bytes_per_step": ndof * 8, "d2h_bytes_per_step": ndof * 8,
                "ms_per_step": e2e_ms, "wall_ms_per_step": wall_e2e,
                "call": ("LdgSystem.residual_tangent(state, du) with numpy du -> numpy R "
                         "(the reference's calling convention)" if world == 1 else
                         "PartitionedLdgSystem.tangent_dev on the H2D copy of numpy du, D2H of R"),
                "pinned_torch": {"value": world * ndof / (e2e_pin_ms * 1e-3) / 1e9,
                                 "ms_per_step": e2e_pin_ms, "wall_ms_per_step": wall_pin}},
        "roofline": {"bound": "hbm", "kernel": p1_name,
                     "achieved": ach_p1, "peak": hbm, "unit": "GB/s",
                     "frac": ach_p1 / hbm, "traffic": traffic.get("pass1"),
                     "traffic_source": traffic.get("source"),
                     "algorithmic_bytes_per_dof": bytes_p1 / ndof, "ms": p1,
                     "peak_source": peak_src,
                     # what bounds it instead (same ncu capture): the L1 / shared
                     # pipe, with 8 warps / SM of a 255-register kernel
                     "pipes": {k: traffic.get("pass1_" + k) for k in
                               ("l1tex_busy", "issue_active", "fp64_pipe", "shared_wavefronts")}
                              if traffic.get("pass1_l1tex_busy") is not None else None,
                     "pipes_source": traffic.get("pipes_source")},
        "pass2_roofline": {"kernel": "complete_warp4_kernel (pass 2, shuffle face lift)", "achieved": ach_p2,
                           "frac": ach_p2 / hbm, "algorithmic_bytes_per_dof": bytes_p2 / ndof,
                           "traffic": traffic.get("pass2"), "ms": p2},
        "matvec_roofline": {"achieved": ach_mv, "peak": hbm, "unit": "GB/s",
                            "frac": ach_mv / hbm, "algorithmic_bytes_per_dof": BYTES_MATVEC,
                            "note": "SURVEY 8(d) two-pass accounting (q through HBM)",
                            "target_60pct_gdofs": 0.6 * hbm / BYTES_MATVEC,
                            "fused_bytes_per_dof": (bytes_p1 + bytes_p2) / ndof,
                            "fused_frac": ach_fused / hbm},
        "unfused_reference_structure": None if world > 1 else {
            "ms_per_step": float(np.median(unf_ms)), "mixed_ms": float(np.median(unf_mixed)),
            "gdofs": ndof / (float(np.median(unf_ms)) * 1e-3) / 1e9},
        "gpu_launches": 2 * args.steps,
        "clocks": clk.summary(),
    }
    if world == 1:
        line["fp64"] = fp64_line(p1)
    if world == 1 and not args.no_solve:
        # the solve runs on the bench system right after the matvec timing,
        # before the other workloads fill the caching allocator
        line["solve"] = {"metric": "Newton-GMRES time to solution (s), config 3, block-Jacobi, "
                                   "acceptance flags", "dofs": ndof,
                         "gpu": run_solve(s)}
        if not args.no_cpu_baseline:
            line["solve"]["cpu_oracle_small"] = {"n": 3, **cpu_solve(3)}
    if world > 1 and solve_line is not None:
        line["solve"] = solve_line
    if strong_line is not None:
        line["strong_scaling"] = strong_line
    if world == 1 and not args.no_tet:
        line["tet"] = tet_line(hbm)
    if world == 1 and not args.no_nonlinear:
        line["nonlinear"] = nonlinear_lines(hbm, cpu=not args.no_cpu_baseline)
    if world == 1 and not args.no_config5:
        line["config5"] = config5_lines(hbm)
    if not args.no_cpu_baseline:
        ts, nd_cpu, cores, kind = reference_times(CPU_SAMPLE_N, 3, 1, ref_procs())
        v = nd_cpu / float(np.median(ts)) / 1e9
        line["cpu_baseline"] = {
            "value": v, "unit": "GDOF/s", "cores": cores, "kind": kind,
            "sample": f"{cores} processes x {nd_cpu // cores}-DOF hex p=3 Poisson tangent (n="
                      f"{CPU_SAMPLE_N}) of " + ("ldgkit (unmodified, baseline/_ref)"
                                                 if kind == "reference" else "the oracle port")
                      + ", median of 3 synchronised steps after 1 warm-up"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--elems", dest="n", type=int, default=N_ELEM,
                    help="hexes per direction per rank (default 54 -> 10,077,696 DOFs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fused", type=int, default=None,
                    help="A/B: 1 / 0 forces the one-launch operator on / off (ldg_set_option 'fused')")
    ap.add_argument("--no-tet", action="store_true",
                    help="skip the config-3 tet variant (44^3 Kuhn tets, dense kernels)")
    ap.add_argument("--no-config5", action="store_true",
                    help="skip the config-5 sweep (conv-diff periodic, hex p = 1..5, ~10M DOFs each)")
    ap.add_argument("--no-solve", action="store_true",
                    help="skip the Newton-GMRES time-to-solution measurement")
    ap.add_argument("--no-nonlinear", action="store_true",
                    help="skip the generated-kernel (configs 2 / 4) throughput lines")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # self-launch one rank per GPU (the driver's torchrun command, same flags)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
        # LDG_DIST_BACKEND=gloo lets several ranks share one GPU (testing only)
        dist.init_process_group(os.environ.get("LDG_DIST_BACKEND", "nccl"))
    run_b200(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
