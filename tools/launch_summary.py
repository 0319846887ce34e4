"""Per-kernel totals and shares of an ncu launch list
(--metrics gpu__time_duration.sum --csv):  python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[h], rows[h + 1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in data:
    k = r[ki].split("(")[0]
    tot[k] += float(r[vi].replace(",", ""))
    cnt[k] += 1
skip = ("at::", "peak_butterfly")
ours = {k: v for k, v in tot.items() if not any(s in k for s in skip)}
s = sum(ours.values())
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'share':>6s}  (path kernels only; cold-cache, serialised)")
for k, v in sorted(ours.items(), key=lambda x: -x[1]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {v / 1e3:10.1f} {100 * v / s:5.1f}%")
