"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch list: per-kernel mean and share."""
import collections, csv, sys
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
only_rs = "--all" not in sys.argv  # default: this library's kernels only (the step)
rows = list(csv.reader(lines))
h = rows[0]; iN = h.index("Kernel Name"); iV = h.index("Metric Value"); iU = h.index("Metric Unit")
t = collections.OrderedDict()
for r in rows[1:]:
    k = r[iN].split('(')[0].replace('<unnamed>::', '').replace('void ', '')
    if only_rs and not k.startswith('rs::'):
        continue
    v = float(r[iV]) * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(r[iU], 1.0)
    t.setdefault(k, []).append(v)
tot = sum(sum(v) for v in t.values())
print(f"| kernel | launches | mean us | share of step (library kernels) |\n|---|---|---|---|")
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    print(f"| {k} | {len(v)} | {sum(v)/len(v):.1f} | {100*sum(v)/tot:.1f}% |")
