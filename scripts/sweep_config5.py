"""Config 5 (BASELINE.json configs[4]): 3D convection-diffusion tangent
matvec, fully periodic unit cube, hex p = 1..5 at ~10M DOFs each
(p=1 n=108, p=2 n=72, p=3 n=54, p=4 n=43, p=5 n=36).

    python scripts/sweep_config5.py [--reps 20] [--p 1,2,3,4,5]

One JSON line: per p the GDOF/s of J(u)du on one B200 (CUDA events on the
launching stream, L2 flushed between reps), the fused-pass algorithmic
bytes per DOF and the HBM fraction of each, and which pass-1 kernel ran."""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

N_FOR_P = {1: 108, 2: 72, 3: 54, 4: 43, 5: 36}
PERIODIC = [(1, 2, (1.0, 0.0, 0.0)), (3, 4, (0.0, 1.0, 0.0)), (5, 6, (0.0, 0.0, 1.0))]


def run_p(p, reps, hbm):
    import torch
    from paper_2205_07824_b200 import meshgen, model, refelem
    from paper_2205_07824_b200.system import LdgSystem
    n = N_FOR_P[p]
    m = model.builtin_model("convection_diffusion", nd=3, mu=[1.0, 1.0, 1.0, 1.0])
    m.bcs = {}
    t0 = time.time()
    mesh = meshgen.generate_structured([(0.0, 1.0)] * 3, [n] * 3, "hex")
    topo = meshgen.build_face_topology(mesh, PERIODIC)
    s = LdgSystem(m, mesh, topo, refelem.build_master("hex", p))
    setup = time.time() - t0
    shape = (s.n_elements, s.n_nodes, 1)
    du = torch.randn(shape, dtype=torch.float64, device="cuda",
                     generator=torch.Generator(device="cuda").manual_seed(0))
    out, X = torch.empty_like(du), s.scratch()
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for _ in range(3):
        s.tangent_dev(du, out=out, scratch=X)
    st = torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        s.tangent_dev(du, out=out, scratch=X)
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    info = s.tab.finfo
    interior = (info & 3) == 0
    sw, right = (info & 8) > 0, (info & 4) > 0
    exports = int(np.sum(interior & (sw == right)))
    completes = int(np.sum(interior & (sw != right)))
    nfn = s.tab.nfn
    nd_ = s.n_dofs
    bytes_fused = 32 * nd_ + 8 * (exports + completes) * nfn
    return {"p": p, "n": n, "dofs": nd_, "ms": ms, "gdofs": nd_ / ms / 1e6,
            "fused_bytes_per_dof": bytes_fused / nd_,
            "fused_frac_hbm": bytes_fused / (ms * 1e-3) / 1e9 / hbm,
            "survey_72B_frac_hbm": 72 * nd_ / (ms * 1e-3) / 1e9 / hbm,
            "pass1_kernel": {1: "plane_g", 2: "plane_g", 3: "plane"}.get(p, "pencil"), "setup_s": round(setup, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--p", default="1,2,3,4,5")
    a = ap.parse_args()
    try:
        hbm = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    except Exception:
        hbm = 6650.0
    rows = [run_p(int(p), a.reps, hbm) for p in a.p.split(",")]
    print(json.dumps({"metric": "config 5: 3D conv-diff periodic tangent matvec GDOF/s, p=1..5",
                      "unit": "GDOF/s", "n_gpus": 1, "hbm_peak_gbs": hbm, "rows": rows}))


if __name__ == "__main__":
    main()
