"""Summarise an ncu report (kernel time, DRAM bytes, pipes, smem wavefronts, stalls)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
idx = {h: i for i, h in enumerate(hdr)}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__shared_mem_per_block_static",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "memory_l1_wavefronts_shared_ideal",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum"]
for r in rows[2:]:
    print("=====", r[idx["Kernel Name"]][:90])
    for w in want:
        if w in idx:
            print(f"  {w:62s} {r[idx[w]]:>16s} {units[idx[w]]}")
    st = [(h[len('smsp__average_warp_latency_issue_stalled_'):] if h.startswith('smsp__average_warp_latency_issue_stalled_') else h, r[i])
          for h, i in idx.items() if h.startswith("smsp__warp_issue_stalled_") and h.endswith("_per_warp_active.pct")]
    st = sorted(((h.replace("smsp__warp_issue_stalled_", "").replace("_per_warp_active.pct", ""), float(v or 0)) for h, v in st), key=lambda x: -x[1])[:6]
    print("  top stalls (% of warp-active cycles):", ", ".join(f"{h} {v:.1f}" for h, v in st))
