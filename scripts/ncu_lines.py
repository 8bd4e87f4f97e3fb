"""Per-source-line totals from an ncu report (source page, CUDA + SASS
view): stall samples, instructions, shared wavefronts (excess = bank
conflicts), local (spill) traffic.

    python scripts/ncu_lines.py rep.ncu-rep [top] [kernel-regex]
"""
import csv, io, subprocess, sys

KEYS = ["Warp Stall Sampling (All Samples)", "Instructions Executed", "L1 Wavefronts Shared",
        "L1 Wavefronts Shared Excessive"]


def main(path, top=40, kernel=None):
    cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel:
        cmd += ["--kernel-name", f"regex:{kernel}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    head = rows[hi]
    idx = [head.index(k) for k in KEYS]
    sp = head.index("Address Space") if "Address Space" in head else None
    lines, cur = {}, None
    def num(s):
        try: return float(s.replace(",", ""))
        except ValueError: return 0.0
    fname = ""
    for r in rows[hi + 1:]:
        if r and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            cur = None
            continue
        if len(r) < len(head):
            continue
        if r[0] == "Line No" or not (r[0] == "" or r[0].isdigit()):
            cur = None
            continue
        if r[0]:
            cur = (fname, int(r[0]), r[1].strip()[:80])
            lines.setdefault(cur, [0.0] * (len(KEYS) + 1))
            continue
        if cur is None:
            continue
        acc = lines[cur]
        for j, i in enumerate(idx):
            acc[j] += num(r[i])
        if sp is not None and r[sp] == "Local":
            acc[-1] += num(r[idx[1]])
    tot = [sum(v[j] for v in lines.values()) for j in range(len(KEYS) + 1)]
    print(f"total samples {tot[0]:.0f} inst {tot[1]:.0f} shared wf {tot[2]:.0f} "
          f"excess {tot[3]:.0f} local inst {tot[4]:.0f}")
    print(" samples       inst  shared_wf   excess  local  line")
    for (fn, ln, src), v in sorted(lines.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{v[0]:8.0f} {v[1]:10.0f} {v[2]:9.0f} {v[3]:8.0f} {v[4]:6.0f}  {fn[:12]}:{ln:<5} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40,
         sys.argv[3] if len(sys.argv) > 3 else None)
