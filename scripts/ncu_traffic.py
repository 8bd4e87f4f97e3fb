"""Write profiles/traffic.json: DRAM bytes per launch of the fused pass-1 /
pass-2 kernels from an ncu --set full report of the bench command.

    python scripts/ncu_traffic.py gpurun_out/prof_bench.ncu-rep [source-note]
"""
import csv
import json
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
idx = {h: i for i, h in enumerate(hdr)}
res = {"source": sys.argv[2] if len(sys.argv) > 2 else rep}


def mb(r, k):
    v = float(r[idx[k]].replace(",", ""))
    u = units[idx[k]]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


for r in rows[2:]:
    name = r[idx["Kernel Name"]]
    b = mb(r, "dram__bytes_read.sum") + mb(r, "dram__bytes_write.sum")
    key = "pass1" if ("plane_kernel" in name or "fused_kernel" in name) else (
        "pass2" if "complete" in name else name[:40])
    res.setdefault(key, b)
    res.setdefault(key + "_kernel", name[:80])
    if key == "pass1" and "pass1_l1tex_busy" not in res:
        # what bounds pass 1 instead of DRAM (bench.py roofline.pipes)
        f = lambda k: float(r[idx[k]].replace(",", ""))
        res["pass1_l1tex_busy"] = f("l1tex__throughput.avg.pct_of_peak_sustained_active") / 100
        res["pass1_issue_active"] = f("smsp__issue_active.avg.pct_of_peak_sustained_active") / 100
        res["pass1_fp64_pipe"] = f("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active") / 100
        res["pass1_shared_wavefronts"] = f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
        res["pipes_source"] = res["source"] + " (l1tex__throughput, smsp__issue_active, " \
            "sm__inst_executed_pipe_fp64, l1tex__data_pipe_lsu_wavefronts_mem_shared)"
json.dump(res, open("profiles/traffic.json", "w"), indent=1)
print(json.dumps(res))
