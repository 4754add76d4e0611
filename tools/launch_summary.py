"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel device time and share.  Usage: launch_summary.py launches.csv [header]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
cols = rows[hdr]
ki, vi, ui = cols.index("Kernel Name"), cols.index("Metric Value"), cols.index("Metric Unit")
tot = collections.Counter()
cnt = collections.Counter()
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
    name = r[ki]
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
print(f"# total kernel time {T:.1f} ms over {sum(cnt.values())} launches\n")
print(f"{'ms':>10} {'share':>6} {'launches':>8}  kernel")
for k, v in tot.most_common():
    print(f"{v:10.2f} {v / T:6.1%} {cnt[k]:8d}  {k}")
