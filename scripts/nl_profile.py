"""Profile helper: run the NS3D tangent a few times, dump the generated
source as ./ldg_nl.cu (the name NVRTC compiled it under) for ncu's source view."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np, torch
from cases import TRANSIENT_CASES, build_case, b200_setup, case_state
from paper_2205_07824_b200.system import LdgSystem
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
spec = dict(TRANSIENT_CASES["ns3d_tgv_hex_p2_dirk11"], counts=[n] * 3, p=3,
            state=([1.0, 0.2, -0.1, 0.15, 25.0], 0.05))
s = LdgSystem(*build_case(spec, *b200_setup()))
Path("ldg_nl.cu").write_text(s.nl.src)
shape = (s.n_elements, s.n_nodes, s.ncu)
u = torch.as_tensor(case_state(spec, *shape, 1), device="cuda")
du = torch.randn(shape, dtype=torch.float64, device="cuda")
for _ in range(4):
    s.tangent_dev(du, base=u)
torch.cuda.synchronize()
print("ok")
