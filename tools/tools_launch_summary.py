"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hi]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("vr::(anonymous namespace)::", "").replace("void ", "")
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    v_us = v / 1e3 if u in ("nsecond", "ns") else v * 1e3 if u in ("msecond", "ms") else v
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v_us
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':55s} {'launches':>8s} {'avg_us':>9s} {'share':>6s}")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:55]:55s} {c:8d} {t / c:9.1f} {100 * t / tot:5.1f}%")
print(f"total launches {sum(a[0] for a in agg.values())}, total {tot / 1e3:.2f} ms (cold-cache, serialised)")
