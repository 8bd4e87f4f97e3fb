"""Summarise an `ncu --set full` report: the metrics DESIGN.md quotes per
kernel plus the top warp-stall reasons.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN_ncu_vX_summary.txt
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_static",
    "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "local_load_requests",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum",
]
STALL = "smsp__average_warp_latency_issue_stalled_"
STALL2 = "smsp__warp_issue_stalled_"


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(head)}
    for r in data:
        name = r[col["Kernel Name"]]
        print(f"===== {name[:100]}")
        for m in METRICS:
            if m in col:
                print(f"  {m:<66} {r[col[m]]:>20} {units[col[m]]}")
        stalls = []
        pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
        for h, i in col.items():
            if h.startswith(pre) and h.endswith(suf):
                try:
                    stalls.append((float(r[i].replace(",", "")), h[len(pre):-len(suf)]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("  top stalls (warps stalled per issued instruction): " +
              ", ".join(f"{n} {v:.2f}" for v, n in stalls[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
