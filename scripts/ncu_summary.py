"""Summarise ncu output (read here, no GPU needed) into profiles/.

usage: python scripts/ncu_summary.py <prof.ncu-rep> <launches.csv> <out-prefix> <workload-key>
writes <out-prefix>.md (launch list shares + key metrics + top stalls) and merges the
closure kernel's dram bytes per launch into profiles/closure_kernel_traffic.json.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

NCU = "ncu"


def raw_metrics(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def details(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res = {}
    for r in rows[1:]:
        if len(r) >= 15 and r[13]:
            res[(r[11], r[12])] = (r[14], r[13])
    return res


def top_stalls(rep, n=12):
    out = subprocess.run([NCU, "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for idx, r in enumerate(rows[2:]):
        try:
            data.append((int(r[i_s]), idx, r[i_src].strip()))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    return [(100.0 * s / tot, idx, src) for s, idx, src in sorted(data, reverse=True)[:n]], tot


def launches(path):
    rows = list(csv.reader(open(path)))
    k = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[k]
    i_name, i_metric, i_val = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[k + 1:]:
        if len(r) > i_val and r[i_metric] == "gpu__time_duration.sum":
            v = float(r[i_val].replace(",", ""))
            unit = r[i_val - 1] if i_val > 0 else ""
            agg[r[i_name].split("(")[0]][0] += 1
            agg[r[i_name].split("(")[0]][1] += v
    return agg


def main():
    rep, lcsv, prefix, key = sys.argv[1:5]
    m = raw_metrics(rep)
    d = details(rep)
    st, tot = top_stalls(rep)
    L = launches(lcsv)
    rd = float(m["dram__bytes_read.sum"][0]) * (1e6 if m["dram__bytes_read.sum"][1] == "Mbyte" else
                                                  1e9 if m["dram__bytes_read.sum"][1] == "Gbyte" else
                                                  1e3 if m["dram__bytes_read.sum"][1] == "Kbyte" else 1)
    wr = float(m["dram__bytes_write.sum"][0]) * (1e6 if m["dram__bytes_write.sum"][1] == "Mbyte" else
                                                   1e9 if m["dram__bytes_write.sum"][1] == "Gbyte" else
                                                   1e3 if m["dram__bytes_write.sum"][1] == "Kbyte" else 1)
    lines = [f"# ncu summary — {key}", "",
             f"source: `{os.path.basename(rep)}` (ncu --set full --clock-control none, one closure_kernel launch) and "
             f"`{os.path.basename(lcsv)}` (--metrics gpu__time_duration.sum, every launch of a 2-step bench run; "
             "cold-cache, serialised — compare shares, not absolutes)", "",
             "## Launch list (device time by kernel)", "", "| kernel | launches | total | share |", "|---|---|---|---|"]
    T = sum(v[1] for v in L.values()) or 1
    for name, (c, t) in sorted(L.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{name}` | {c} | {t:.1f} | {100 * t / T:.1f}% |")
    lines += ["", "(units of gpu__time_duration.sum as reported by ncu: ns or us per the CSV)", "",
              "## profiled kernel (full set)", "", "| metric | value |", "|---|---|"]
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
              "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
              "lts__t_sectors_srcunit_tex_op_atom.sum", "smsp__inst_executed.sum",
              "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
              "lts__t_bytes.sum", "l1tex__t_bytes.sum"]:
        if k in m:
            lines.append(f"| {k} | {m[k][0]} {m[k][1]} |")
    for (sec, name), (v, u) in d.items():
        if name in ("L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Achieved Occupancy", "Eligible Warps Per Scheduler",
                    "DRAM Throughput", "Mem Busy"):
            lines.append(f"| {sec}: {name} | {v} {u} |")
    lines += ["", f"## Top SASS stall sites ({tot} samples)", "", "| share | idx | SASS |", "|---|---|---|"]
    for share, idx, src in st:
        lines.append(f"| {share:.1f}% | {idx} | `{src}` |")
    with open(prefix + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    tj = os.path.join(os.path.dirname(prefix), "closure_kernel_traffic.json")   # per-workload dominant kernel
    try:
        data = json.load(open(tj))
    except Exception:
        data = {}
    data[key] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "source": os.path.basename(rep)}
    json.dump(data, open(tj, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
