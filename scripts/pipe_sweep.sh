#!/bin/bash
for c in 8 16 32; do
  LDG_PIPE_CHUNKS=$c python - <<'PY'
import sys, time, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import torch
from bench import build_problem
from paper_2205_07824_b200.system import LdgSystem, SolverState
m, mesh, topo, master = build_problem(54)
s = LdgSystem(m, mesh, topo, master)
h = torch.randn((s.n_elements, s.n_nodes, 1), dtype=torch.float64).pin_memory()
st = SolverState(u=h, q=None, w=None, t=0.0)
for _ in range(5): out = s.residual_tangent(st, h)[0]
torch.cuda.synchronize()
t0 = time.perf_counter(); k = 20
for _ in range(k): out = s.residual_tangent(st, h)[0]
dt = (time.perf_counter() - t0) / k
print(f"chunks {os.environ['LDG_PIPE_CHUNKS']}: e2e {dt*1e3:.3f} ms  {s.n_dofs/dt/1e9:.2f} GDOF/s")
PY
done
