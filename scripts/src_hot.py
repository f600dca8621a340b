"""Per-CUDA-line instruction/stall shares from `ncu --page source --print-source cuda,sass --csv`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur = None; hdr = None; out = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path": cur = r[1].split('/')[-1]; continue
    if len(r) >= 2 and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8 or r[2] != "-": continue
    try: ins = float(r[7]); st = float(r[4])
    except ValueError: continue
    out.append((ins, st, cur, r[0], r[1][:110]))
tot = sum(o[0] for o in out) or 1; tots = sum(o[1] for o in out) or 1
print(f"total warp instrs {tot:.3g}, stall samples {tots:.3g}")
key = 1 if (len(sys.argv) > 3 and sys.argv[3] == "stall") else 0
for o in sorted(out, key=lambda o: -o[key])[:n]:
    print(f"{100*o[0]/tot:5.1f}% {100*o[1]/tots:5.1f}%  {o[2]}:{o[3]}  {o[4]}")
