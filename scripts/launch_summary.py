"""Per-kernel totals of an ncu --csv launch list (time, share, DRAM bytes): python scripts/launch_summary.py f.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = defaultdict(lambda: defaultdict(float))
cnt = defaultdict(int)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    k = d["Kernel Name"].split("(")[0][:60]
    v = float(d["Metric Value"].replace(",", ""))
    agg[k][d["Metric Name"]] += v
    if d["Metric Name"] == "gpu__time_duration.sum":
        cnt[k] += 1
tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'ms':>9s} {'share':>6s} {'DRAM GB':>8s} {'GB/s':>7s}")
for k, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    t = a["gpu__time_duration.sum"]
    by = a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)
    print(f"{k:60s} {cnt[k]:8d} {t / 1e6:9.3f} {t / tot:6.3f} {by / 1e9:8.2f} {by / t if t else 0:7.1f}")
