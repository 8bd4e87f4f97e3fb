"""Where the e2e time goes: pinned H2D / D2H bandwidth vs the drop-in call."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import torch
from bench import build_problem
from paper_2205_07824_b200.system import LdgSystem, SolverState

m, mesh, topo, master = build_problem(54)
s = LdgSystem(m, mesh, topo, master)
shape = (s.n_elements, s.n_nodes, 1)
h = torch.randn(shape, dtype=torch.float64).pin_memory()
d = torch.empty(shape, dtype=torch.float64, device="cuda")
o = torch.empty(shape, dtype=torch.float64).pin_memory()
st = torch.cuda.current_stream()
def ev(fn, n=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(n): fn()
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
nb = h.numel() * 8
t = ev(lambda: d.copy_(h, non_blocking=True)); print(f"H2D {t:.3f} ms  {nb/t/1e6:.1f} GB/s")
t = ev(lambda: o.copy_(d, non_blocking=True)); print(f"D2H {t:.3f} ms  {nb/t/1e6:.1f} GB/s")
s2 = torch.cuda.Stream()
def both():
    d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        o.copy_(d2, non_blocking=True)
    st.wait_stream(s2)
d2 = torch.empty_like(d)
t = ev(both); print(f"H2D||D2H {t:.3f} ms  {2*nb/t/1e6:.1f} GB/s total")
t = ev(lambda: torch.empty(shape, dtype=torch.float64, pin_memory=True)); print(f"pinned alloc {t:.3f} ms")
state = SolverState(u=h, q=None, w=None, t=0.0)
t0 = time.perf_counter(); n = 10
for _ in range(n): r = s.residual_tangent(state, h)[0]
print(f"residual_tangent(host torch) wall {(time.perf_counter()-t0)/n*1e3:.3f} ms")
t = ev(lambda: s.tangent_dev(d)); print(f"tangent_dev {t:.3f} ms")
# step-by-step wall times of the drop-in call
import paper_2205_07824_b200._lib as L
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dd, dev = s._dev(h)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    R = s.tangent_dev(dd.reshape(shape))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    s._check_nan("flux")
    t3 = time.perf_counter()
    out = s._ret(R, dev)
    t4 = time.perf_counter()
    print(f"_dev {1e3*(t1-t0):.3f}  tangent {1e3*(t2-t1):.3f}  check_nan {1e3*(t3-t2):.3f}  _ret {1e3*(t4-t3):.3f} ms")
