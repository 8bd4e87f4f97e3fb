"""Where the first (cold) config-3 solve of a process spends its extra time
over a warm one: block-Jacobi build phases and the GMRES start-up, with
synchronised wall-clock marks."""
import sys
import time
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import torch
from bench import build_problem
from paper_2205_07824_b200 import solver
from paper_2205_07824_b200.driver import _steady_fns, run_steady
from paper_2205_07824_b200.system import LdgSystem

n = int(sys.argv[1]) if len(sys.argv) > 1 else 54
s = LdgSystem(*build_problem(n))
torch.cuda.synchronize()
T = {}


def tm(name, fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    T.setdefault(name, []).append(round(time.perf_counter() - t, 4))
    return r


orig = solver._block_classes
solver._block_classes = lambda m, **k: tm("bj_classes", lambda: orig(m, **k))
orig_tiles = solver.class_tiles
solver.class_tiles = lambda *a: tm("bj_tiles", lambda: orig_tiles(*a))
for rep in range(2):
    st = tm("init", s.interpolate_initial_dev)
    res, tan = _steady_fns(s)
    u0 = st.u.reshape(-1)
    from paper_2205_07824_b200.driver import build_pde_block_jacobi
    M = tm("bj_build", lambda: build_pde_block_jacobi(s, res, tan, u0))
    tm("bj_apply_first", lambda: M.apply(u0))
    out = tm("run_steady", lambda: run_steady(s, precond="block_jacobi", orth="dcgs2"))
    T.setdefault("run_steady_split", []).append({k: round(v, 3) for k, v in out[2].items()
                                                 if isinstance(v, float)})
print(T)
