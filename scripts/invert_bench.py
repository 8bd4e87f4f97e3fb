"""Time ldg_bj_invert on config-3-sized batches (157464 blocks of 64 x 64)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2205_07824_b200 import _lib
lib = _lib.load()
nb, bs = 157464, 64
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn((nb, bs, bs), dtype=torch.float64, device="cuda", generator=g)
A += 2 * bs * torch.eye(bs, dtype=torch.float64, device="cuda")
inv = torch.empty_like(A)
sh = torch.empty(nb, dtype=torch.int32, device="cuda")
ts = []
for _ in range(4):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.check(lib.ldg_bj_invert(nb, bs, _lib.ptr(A), _lib.ptr(inv), _lib.ptr(sh), _lib.stream_ptr()), "inv")
    b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
I = torch.bmm(A[:64], inv[:64].transpose(1, 2))
print("invert ms", [round(t, 2) for t in ts], "max |A inv - I|", float((I - torch.eye(bs, device="cuda", dtype=torch.float64)).abs().max()))
