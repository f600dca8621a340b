"""Top SASS instructions by stall samples / executed count from an ncu source page CSV (--print-source sass)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
def f(r, k):
    try: return float(r[ci[k]])
    except: return 0.0
tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
tot_i = sum(f(r, "Instructions Executed") for r in data)
print(f"total stall samples {tot_s:.0f}, warp instrs {tot_i:.0f}")
# opcode histogram
ops = collections.Counter(); stalls = collections.Counter()
for r in data:
    op = r[ci["Source"]].split()[0] if r[ci["Source"]].split() else "?"
    if op.startswith("@"): op = r[ci["Source"]].split()[1]
    op = op.split(".")[0]
    ops[op] += f(r, "Instructions Executed"); stalls[op] += f(r, "Warp Stall Sampling (All Samples)")
print("opcode: instr% stall%")
for op, v in ops.most_common(25):
    print(f"  {op:10s} {100*v/tot_i:5.1f}% {100*stalls[op]/max(tot_s,1):5.1f}%")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print("top stall instructions:")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:n]:
    print(f"  {f(r,'Warp Stall Sampling (All Samples)'):7.0f} {f(r,'Instructions Executed'):9.0f}  {r[ci['Address']]} {r[ci['Source']][:90]}")
