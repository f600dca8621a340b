"""Summarise an ncu --set full report: key metrics per kernel -> markdown (+ optional traffic JSON).

usage: python scripts/ncu_summary.py REPORT.ncu-rep OUT.md [--traffic OUT.json --pixels-per-launch P --map kernel_regex=call ...]
"""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    (("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
      "dram__throughput.avg.pct_of_peak_sustained_elapsed"), "dram %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ %"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem confl"),
    ("smsp__inst_executed_op_global_red.sum", "red inst"),
    ("lts__t_sectors_op_red.sum", "L2 red sect"),
    ("lts__t_sectors_op_atom.sum", "L2 atom sect"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "smem atom wavefr"),
]
# extra counters to request with --set full (scripts/gpurun_prof.sh)
EXTRA_METRICS = ",".join(["smsp__inst_executed_op_global_red.sum", "lts__t_sectors_op_red.sum",
                          "lts__t_sectors_op_atom.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
                          "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"])


def load(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True,
                                  stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def stalls(hdr, r, k=3):
    vals = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                vals.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    vals.sort(reverse=True)
    tot = sum(v for v, _ in vals) or 1.0
    return ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in vals[:k])


def main():
    rep, outmd = sys.argv[1], sys.argv[2]
    args = sys.argv[3:]
    hdr, units, data = load(rep)
    col = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu summary of `{rep.split('/')[-1]}`", "",
             "| kernel | " + " | ".join(n for _, n in KEYS) + " | top stalls |",
             "|---" * (len(KEYS) + 2) + "|"]
    per_kernel = {}
    for r in data:
        name = r[col["Kernel Name"]]
        short = re.sub(r"\(.*", "", name).replace("unnamed>::", "").replace("void ", "")
        cells = []
        for k, _ in KEYS:
            ks = k if isinstance(k, tuple) else (k,)
            hit = next((kk for kk in ks if kk in col), None)
            if hit is not None:
                u = units[col[hit]]
                cells.append(f"{r[col[hit]]} {u}".strip())
            else:
                cells.append("-")
        lines.append(f"| {short} | " + " | ".join(cells) + f" | {stalls(hdr, r)} |")
        try:
            rd = float(r[col["dram__bytes_read.sum"]])
            wr = float(r[col["dram__bytes_write.sum"]])
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            su = scale.get(units[col["dram__bytes_read.sum"]], 1)
            sw = scale.get(units[col["dram__bytes_write.sum"]], 1)
            per_kernel.setdefault(short, []).append(rd * su + wr * sw)
        except (KeyError, ValueError):
            pass
    with open(outmd, "w") as f:
        f.write("\n".join(lines) + "\n")
    if "--traffic" in args:
        out = args[args.index("--traffic") + 1]
        px = float(args[args.index("--pixels-per-launch") + 1])
        maps = [a.split("=", 1) for a in args if "=" in a and not a.startswith("--")]
        res = {"source": rep.split("/")[-1], "pixels_per_launch": px}
        for rx, call in maps:
            tot = sum(sum(v) / len(v) for k, v in per_kernel.items() if re.search(rx, k))
            res[call] = {"dram_bytes": tot, "per_pixel": tot / px, "kernels": rx}
        with open(out, "w") as f:
            json.dump(res, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
