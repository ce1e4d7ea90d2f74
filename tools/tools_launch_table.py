"""Summarise an `ncu --metrics gpu__time_duration.sum,... --csv --log-file X` launch list:
per kernel: launches, total / average time, share, DRAM bytes read per launch.
    python tools/tools_launch_table.py launches.csv"""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(dict)
names = {}
for r in rows[1:]:
    if len(r) < len(h):
        continue
    per[r[iid]][r[im]] = float(r[iv].replace(",", "")) if r[iv] else 0.0
    names[r[iid]] = r[ik].split("(")[0][:60]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, d in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0.0)
    a[2] += d.get("dram__bytes_read.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{len(per)} launches, {tot / 1e6:.2f} ms total")
print("| kernel | launches | total ms | share | avg us | DRAM read MB/launch |")
print("|---|---|---|---|---|---|")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| {k} | {a[0]} | {a[1] / 1e6:.2f} | {100 * a[1] / tot:.1f}% | {a[1] / a[0] / 1e3:.1f} | {a[2] / a[0] / 1e6:.1f} |")
