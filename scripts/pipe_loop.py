import sys, time
from pathlib import Path
R_ = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(R_)); sys.path.insert(0, str(R_ / "tests"))
import torch
from bench import build_problem
from paper_2205_07824_b200.system import LdgSystem, SolverState
m, mesh, topo, master = build_problem(54)
s = LdgSystem(m, mesh, topo, master)
h = torch.randn((s.n_elements, s.n_nodes, 1), dtype=torch.float64).pin_memory()
st = SolverState(u=h, q=None, w=None, t=0.0)
ts = []
for i in range(12):
    t0 = time.perf_counter()
    out = s.residual_tangent(st, h)[0]
    ts.append((time.perf_counter() - t0) * 1e3)
print("per-call wall ms:", [round(x, 2) for x in ts])
ts = []
outs = []
for i in range(6):
    t0 = time.perf_counter()
    outs.append(s.residual_tangent(st, h)[0])
    ts.append((time.perf_counter() - t0) * 1e3)
print("keeping results:", [round(x, 2) for x in ts])
