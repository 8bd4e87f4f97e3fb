"""Where the config-3 steady solve spends its time: torch.profiler over
run_steady (CUDA kernel totals vs wall), n=54 hex p=3 by default.

    python scripts/solve_profile.py [--n 54] [--orth cgs2]
"""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "scripts"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=54)
    ap.add_argument("--orth", default="cgs2")
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    from solve_bench import build
    from paper_2205_07824_b200.driver import run_steady
    from paper_2205_07824_b200.system import LdgSystem
    s = LdgSystem(*build(a.n))
    run_steady(s, precond="block_jacobi", orth=a.orth)          # warm-up (JIT, allocations)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        _, stats, tm = run_steady(s, precond="block_jacobi", orth=a.orth)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    print("wall", wall, tm, "gmres", stats.total_gmres_iters)
    ka = prof.key_averages()
    cuda_total = sum(k.self_device_time_total for k in ka) / 1e6
    print(f"CUDA kernel time total {cuda_total:.3f} s")
    print(ka.table(sort_by="self_device_time_total", row_limit=15, max_name_column_width=60))
    print(ka.table(sort_by="self_cpu_time_total", row_limit=15, max_name_column_width=60))


if __name__ == "__main__":
    main()
