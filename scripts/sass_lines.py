"""Aggregate an ncu SASS source page (csv) by CUDA source line using nvdisasm -g line info.

usage: python scripts/sass_lines.py <src_sass.csv> <disasm.sass> <mangled kernel> [top]
"""
import csv, re, sys, collections

csv_path, sass_path, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lines = open(sass_path).read().split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith(f".text.{kern}:"))
off2line, cur = {}, None
for l in lines[start + 1:]:
    if l.startswith("//----"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csv_path)))
hdr = rows[1]
ia, ie, isamp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
base = int(rows[2][ia], 16)
ins, smp = collections.Counter(), collections.Counter()
tot_i = tot_s = 0
for r in rows[2:]:
    if len(r) <= ie or not r[ia].startswith("0x"):
        continue
    off = int(r[ia], 16) - base
    key = off2line.get(off)
    i, s = int(r[ie] or 0), int(r[isamp] or 0)
    ins[key] += i
    smp[key] += s
    tot_i += i
    tot_s += s
print(f"total warp instructions {tot_i}  stall samples {tot_s}")
print("by instructions:")
for k, v in ins.most_common(top):
    print(f"  {v:10d} {100*v/tot_i:5.1f}%  samples {100*smp[k]/max(tot_s,1):5.1f}%  {k}")
print("by stall samples:")
for k, v in smp.most_common(top):
    print(f"  {100*v/max(tot_s,1):5.1f}%  inst {ins[k]:10d}  {k}")

# regions (engine.cu line ranges) given as name=lo-hi arguments after [top]
regions = [a for a in sys.argv[5:] if "=" in a]
if regions:
    print("by region:")
    for spec in regions:
        name, rng = spec.split("=")
        lo, hi = map(int, rng.split("-"))
        ti = sum(v for k, v in ins.items() if k and k[0] == "engine.cu" and lo <= k[1] <= hi)
        ts = sum(v for k, v in smp.items() if k and k[0] == "engine.cu" and lo <= k[1] <= hi)
        print(f"  {name:14s} inst {ti:10d} {100*ti/tot_i:5.1f}%  samples {100*ts/max(tot_s,1):5.1f}%")
    other = {k: v for k, v in ins.items() if not k or k[0] != "engine.cu"}
    print("  non-engine.cu inst", sum(other.values()))
