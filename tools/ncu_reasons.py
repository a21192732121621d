"""Per-source-line warp-stall breakdown by reason (ncu --page source --print-source cuda,sass csv)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 20
names = ["stall_wait", "stall_long_sb", "stall_short_sb", "stall_math", "stall_mio", "stall_lg", "stall_barrier",
         "stall_selected", "stall_branch_resolving", "stall_dispatch", "stall_not_selected", "stall_no_inst"]
hdr = None; cur = ""
agg = collections.defaultdict(lambda: collections.Counter()); src = {}
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = {c: j for j, c in enumerate(r)}; continue
    if hdr is None: continue
    try: ln = int(r[0])
    except: continue
    for nm in names:
        try: agg[(cur, ln)][nm] += float(r[hdr[nm]])
        except: pass
    src[(cur, ln)] = r[1]
tot = collections.Counter()
for c in agg.values(): tot.update(c)
T = sum(tot.values())
print("totals:", {k: f"{100*v/T:.1f}%" for k, v in tot.most_common()})
lines = sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:topn]
for (f, ln), c in lines:
    s = sum(c.values())
    top = ", ".join(f"{k[6:]}={100*v/T:.1f}" for k, v in c.most_common(3) if v > 0)
    print(f"{100*s/T:5.1f}% {f}:{ln:<4} [{top}] {src[(f, ln)][:70]}")
