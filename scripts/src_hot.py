"""Per-CUDA-line instruction/stall shares from `ncu --page source --print-source cuda,sass --csv`
(lines aggregated over the report's launches).  usage: src_hot.py CSV [N] [stall]"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur = None; hdr = None
agg = collections.OrderedDict()
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": cur = r[1].split('/')[-1]; continue
    if len(r) >= 2 and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8 or r[2] != "-": continue
    try: ins = float(r[7]); st = float(r[4])
    except ValueError: continue
    k = (cur, r[0])
    a = agg.setdefault(k, [0.0, 0.0, r[1][:110]])
    a[0] += ins; a[1] += st
tot = sum(v[0] for v in agg.values()) or 1; tots = sum(v[1] for v in agg.values()) or 1
print(f"total warp instrs {tot:.3g}, stall samples {tots:.3g}")
key = 1 if (len(sys.argv) > 3 and sys.argv[3] == "stall") else 0
for (f, ln), v in sorted(agg.items(), key=lambda kv: -kv[1][key])[:n]:
    print(f"{100*v[0]/tot:5.1f}% {100*v[1]/tots:5.1f}%  {f}:{ln}  {v[2]}")
