import sys, time, torch
sys.path.insert(0, '.')
sys.path.insert(0, 'scripts')
from solve_bench import build
from paper_2205_07824_b200.system import LdgSystem
from paper_2205_07824_b200.solver import _WS, vecops
s = LdgSystem(*build(54))
torch.cuda.synchronize()
t0 = time.perf_counter(); ws = _WS.get(250, s.n_dofs, torch.device("cuda"), need_z=False); torch.cuda.synchronize(); t1 = time.perf_counter()
ws.V.fill_(0.0); torch.cuda.synchronize(); t2 = time.perf_counter()
print("alloc", t1 - t0, "first touch", t2 - t1)
