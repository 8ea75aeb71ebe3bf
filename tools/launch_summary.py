"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: launches, median time and
share of the total per kernel (cold-cache, serialised launches: compare shares, not absolutes)."""
import collections
import csv
import statistics
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
t = collections.defaultdict(list)
for r in rows[1:]:
    if r[iv].replace(".", "").replace(",", "").isdigit():
        t[r[ik]].append(float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0))
tot = sum(sum(v) for v in t.values())
print(f"{'kernel':70s} launches  median_us   share")
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:70]:70s} {len(v):8d} {statistics.median(v):10.2f} {sum(v) / tot * 100:6.1f}%")
