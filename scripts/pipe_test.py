import sys, time
from pathlib import Path; R_ = Path(__file__).resolve().parent.parent; sys.path.insert(0, str(R_)); sys.path.insert(0, str(R_ / "tests"))
import numpy as np, torch
from bench import build_problem
from paper_2205_07824_b200.system import LdgSystem, SolverState
for n in (12, 54):
    m, mesh, topo, master = build_problem(n)
    s = LdgSystem(m, mesh, topo, master)
    shape = (s.n_elements, s.n_nodes, 1)
    h = torch.randn(shape, dtype=torch.float64).pin_memory()
    st = SolverState(u=h, q=None, w=None, t=0.0)
    J = s.residual_tangent(st, h)[0]
    Jd = s.tangent_dev(h.cuda()).cpu()
    R = s.residual(st)[0]; Rd = s.residual_dev(h.cuda()).cpu()
    print(n, s._pipe_plan()[1], float((J - Jd).abs().max()), float((R - Rd).abs().max()))
    torch.cuda.synchronize()
    for _ in range(3): s.residual_tangent(st, h)
    t0 = time.perf_counter(); k = 10
    for _ in range(k): out = s.residual_tangent(st, h)[0]
    dt = (time.perf_counter() - t0) / k
    print(f"n={n} e2e wall {dt*1e3:.3f} ms  {s.n_dofs/dt/1e9:.2f} GDOF/s")
# device-side timing of the pipeline vs allocation overhead
import paper_2205_07824_b200.system as S
orig = torch.empty
t_alloc = []
def timed_empty(*a, **k):
    t0 = time.perf_counter(); r = orig(*a, **k); t_alloc.append((time.perf_counter() - t0, k.get("pin_memory", False))); return r
torch.empty = timed_empty
for _ in range(5): out = s.residual_tangent(st, h)[0]
torch.empty = orig
print("allocs (ms, pinned):", [(round(a*1e3, 3), p) for a, p in t_alloc[-6:]])
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record(); out = s.residual_tangent(st, h)[0]; ev1.record(); torch.cuda.synchronize()
print(f"device span {ev0.elapsed_time(ev1):.3f} ms")
t0 = time.perf_counter(); out = s.residual_tangent(st, h)[0]; print(f"one call wall {(time.perf_counter()-t0)*1e3:.3f} ms")
