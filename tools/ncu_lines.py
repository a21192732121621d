"""Aggregate ncu warp-stall samples per CUDA source line (ncu --page source --print-source cuda,sass)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
agg = collections.Counter(); src = {}
cur_file = ""
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; i_s = hdr.index("Warp Stall Sampling (All Samples)"); continue
    if hdr is None or len(r) <= i_s: continue
    try: v = float(r[i_s]); ln = int(r[0])
    except: continue
    agg[(cur_file, ln)] += v; src[(cur_file, ln)] = r[1]
tot = sum(agg.values())
print("total samples", tot)
for (f, ln), v in agg.most_common(topn):
    print(f"{100*v/tot:5.1f}% {f}:{ln:<5} {src[(f, ln)][:100]}")
