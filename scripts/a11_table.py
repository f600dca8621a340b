"""profiles/r2_a11.md from the per-variant ncu CSVs (gpurun_out/r2_a11_v<i>.csv: each holds the
variant's warm-up call and one measured call -- the second half of its kernels is summed)
and the event times (gpurun_out/r2_a11_times.jsonl / r2_a11_times64.jsonl)."""
import csv, json, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed_op_global_red.sum", "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "usecond": 1e-6,
         "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9}
t8 = [json.loads(l) for l in open("gpurun_out/r2_a11_times.jsonl")]
t64 = [json.loads(l) for l in open("gpurun_out/r2_a11_times64.jsonl")]
rows = []
for i, (r8, r64) in enumerate(zip(t8, t64)):
    lines = [l for l in open(f"gpurun_out/r2_a11_v{i}.csv") if l.startswith('"')]
    rr = list(csv.reader(lines))
    hdr = rr[0]
    data = rr[1:]
    iN, iM, iU, iV = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    iID = hdr.index("ID")
    per = {}
    for r in data:
        k = int(r[iID])
        try:
            v = float(r[iV].replace(",", "")) * SCALE.get(r[iU], 1.0)
        except ValueError:
            continue
        per.setdefault(k, {})[r[iM]] = v
    ids = sorted(per)
    ids = ids[len(ids) // 2:]  # the measured call
    tot = {m: sum(per[k].get(m, 0.0) for k in ids) for m in KEYS}
    rows.append((r8, r64, tot))
out = ["# Row a11: scatter vs gather per layer, measured (round 2)", "",
       "configs[4] shapes (STN C=16, warp C=3 smooth flow, bslice 16x16x8), one B200.  Event times:",
       "`scripts/prof_a11.py NB REPS` (median, CUDA events).  Counters: one `ncu --metrics ...` run per",
       "variant (`scripts/prof_a11.py 8 1 <variant>`), the measured call's kernels summed (serialised,",
       "cold-cache); built by `scripts/a11_table.py`.  The paper's rule (PAPER.md:723-733): convert a",
       "scatter to a gather where a bounded inverse exists, else fall back to atomics.", "",
       "| call | variant | ms @8 | ms @64 | ncu kernel ms @8 | DRAM MB @8 | global red inst | L2 red sectors | L2 atom sectors | smem atom wavefronts |",
       "|---|---|---|---|---|---|---|---|---|---|"]
for r8, r64, t in rows:
    out.append(f"| {r8['call']} | {r8['variant']} | {r8['ms']:.3f} | {r64['ms']:.3f} | {t['gpu__time_duration.sum'] * 1e3:.3f} | "
               f"{(t['dram__bytes_read.sum'] + t['dram__bytes_write.sum']) / 1e6:.0f} | "
               f"{t['smsp__inst_executed_op_global_red.sum'] / 1e6:.2f} M | {t['lts__t_sectors_op_red.sum'] / 1e6:.1f} M | "
               f"{t['lts__t_sectors_op_atom.sum'] / 1e6:.1f} M | {t['l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum'] / 1e6:.1f} M |")
out += ["", open("scripts/a11_reading.md").read()]
open("profiles/r2_a11.md", "w").write("\n".join(out) + "\n")
print("\n".join(out[8:]))
