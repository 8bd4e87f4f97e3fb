"""A/B of the host pipeline's chunk count on the config-3 e2e call
(LdgSystem.residual_tangent with numpy in / out and with pinned torch
tensors): python scripts/e2e_chunks.py 6 8 12 16"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch
    import bench
    from paper_2205_07824_b200.system import LdgSystem, SolverState
    m, mesh, topo, master = bench.build_problem(bench.N_ELEM, nx_mult=1)
    for c in [int(x) for x in sys.argv[1:]]:
        LdgSystem.PIPE_CHUNKS = c
        s = LdgSystem(m, mesh, topo, master)
        shape = (s.n_elements, s.n_nodes, 1)
        x = np.random.default_rng(0).normal(size=shape)
        xp = torch.as_tensor(x).pin_memory()
        res = {}
        for name, xh in (("numpy", x), ("pinned", xp)):
            st = SolverState(u=xh, q=None, w=None, t=0.0)
            for _ in range(4):
                out = s.residual_tangent(st, xh)[0]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(20):
                out = s.residual_tangent(st, xh)[0]
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) / 20 * 1e3
            res[name] = (round(ms, 3), round(s.n_dofs / ms / 1e6, 2))
        print(c, res, flush=True)
        del s
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
