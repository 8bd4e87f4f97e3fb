"""Per-stage / per-line stall attribution from an ncu source CSV
(--page source --csv --print-source cuda,sass)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
src = open(sys.argv[2]).read().splitlines()
hdr = rows[2]
ws = hdr.index("Warp Stall Sampling (All Samples)"); ie = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
byline = collections.defaultdict(lambda: [0, 0, collections.Counter()])
cur = None
for r in rows[3:]:
    if len(r) < len(hdr):
        continue
    if r[0] not in ("", "-"):
        try:
            cur = int(r[0])
        except ValueError:
            continue
    if cur is None:
        continue
    try:
        byline[cur][0] += int(r[ws] or 0)
        byline[cur][1] += int(r[ie] or 0)
        for i in stall_cols:
            byline[cur][2][hdr[i][6:]] += int(r[i] or 0)
    except ValueError:
        pass
marks = [(i + 1, l.strip()) for i, l in enumerate(src) if l.strip().startswith("// ----")]
def stage(line):
    st = "pre"
    for ln, t in marks:
        if ln <= line:
            st = t[:60]
    return st
agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for ln, (w, n, c) in byline.items():
    a = agg[stage(ln)]
    a[0] += w; a[1] += n; a[2].update(c)
tw = sum(a[0] for a in agg.values()) or 1
tn = sum(a[1] for a in agg.values()) or 1
for k, (w, n, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    top = ", ".join(f"{h}:{v}" for h, v in c.most_common(3))
    print(f"{100*w/tw:5.1f}% stalls {100*n/tn:5.1f}% inst  {k}  [{top}]")
print()
for ln, (w, n, c) in sorted(byline.items(), key=lambda x: -x[1][0])[:int(sys.argv[3]) if len(sys.argv) > 3 else 15]:
    print(f"{w:6d} {n:10d} L{ln:4d} {src[ln-1].strip()[:90]}")
