import sys, time
sys.path.insert(0, "."); sys.path.insert(0, "scripts")
import torch
import paper_2205_07824_b200.solver as S
from solve_bench import build
from paper_2205_07824_b200.driver import run_steady
from paper_2205_07824_b200.system import LdgSystem
# wrap the VecOps kernels and the operator with synchronized wall timers
tot = {}
def wrap(obj, name):
    f = getattr(obj, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); tot[name] = tot.get(name, 0.0) + time.perf_counter() - t
        return r
    setattr(obj, name, g)
s = LdgSystem(*build(54))
ops = S.vecops(s.device)
for n in ("cgs_dots", "cgs_update", "nrm2", "div", "combine", "dot"):
    wrap(ops, n)
wrap(s, "tangent_dev")
t0 = time.perf_counter()
st, stats, tm = run_steady(s, precond="block_jacobi", orth="cgs2")
print("cold", tm, {k: round(v, 3) for k, v in tot.items()})
tot.clear()
st, stats, tm = run_steady(s, precond="block_jacobi", orth="cgs2")
print("warm", tm, {k: round(v, 3) for k, v in tot.items()})
