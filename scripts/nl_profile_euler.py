"""Profile helper: the config-2 Euler 2D quad p=4 tangent (n=128), a few runs."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import torch
from cases import TRANSIENT_CASES, build_case, b200_setup, case_state
from paper_2205_07824_b200.system import LdgSystem
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
spec = dict(TRANSIENT_CASES["euler2d_vortex_quad_p3_dirk22"], counts=[n] * 2, p=4,
            state=([1.0, 0.2, -0.1, 2.5], 0.05))
s = LdgSystem(*build_case(spec, *b200_setup()))
shape = (s.n_elements, s.n_nodes, s.ncu)
u = torch.as_tensor(case_state(spec, *shape, 1), device="cuda")
du = torch.randn(shape, dtype=torch.float64, device="cuda")
for _ in range(4):
    s.tangent_dev(du, base=u)
torch.cuda.synchronize()
print("ok")
