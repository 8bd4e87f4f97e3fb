"""A/B of the generated 3D kernels' launch shape on the config-4 NS tangent:
threads per element, faces per batch of the face phase, register-capped
blocks per SM (nonlinear.NT_3D / FACE_BATCH_3D / MINB_3D).

    python scripts/nl_ab.py 128,6,3 128,2,3 128,2,4 64,2,5 ...   [--ns-n 32]
    python scripts/nl_ab.py 2d:1 2d:24 2d:32    (config-2 Euler: blocks per SM, nonlinear.MINB_2D_C)"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT / "scripts"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("shapes", nargs="+")
    ap.add_argument("--ns-n", type=int, default=32)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import nl_bench
    from cases import TRANSIENT_CASES
    from paper_2205_07824_b200 import nonlinear
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    ns = dict(TRANSIENT_CASES["ns3d_tgv_hex_p2_dirk11"], counts=[a.ns_n] * 3, p=3,
              state=([1.0, 0.2, -0.1, 0.15, 25.0], 0.05))
    eu = dict(TRANSIENT_CASES["euler2d_vortex_quad_p3_dirk22"], counts=[256] * 2, p=4,
              state=([1.0, 0.2, -0.1, 2.5], 0.05))
    for sh in a.shapes:
        if sh.startswith("2d:"):
            nonlinear.MINB_2D_C = int(sh[3:])
            _, v = nl_bench.run("config2_euler2d_quad_p4", eu, a.reps, peak)
            print(json.dumps({"minb_2d_c": nonlinear.MINB_2D_C,
                              **{k: v[k] for k in ("tangent_gdofs", "residual_gdofs", "attrs") if k in v}}),
                  flush=True)
            continue
        vals = [int(x) for x in sh.split(",")]
        nt, fb, minb = vals[:3]
        nonlinear.LOAD_BATCH = vals[3] if len(vals) > 3 else nonlinear.LOAD_BATCH
        nonlinear.NT_3D, nonlinear.FACE_BATCH_3D, nonlinear.MINB_3D = nt, fb, minb
        _, v = nl_bench.run("config4_ns3d_hex_p3", ns, a.reps, peak)
        print(json.dumps({"nt": nt, "fb": fb, "minb": minb, "load_batch": nonlinear.LOAD_BATCH,
                          **{k: v[k] for k in ("tangent_gdofs", "residual_gdofs", "tangent_ms",
                                               "residual_ms", "tangent_uncached_gdofs",
                                               "base_cache_ms", "attrs")
                             if k in v}}), flush=True)


if __name__ == "__main__":
    main()
