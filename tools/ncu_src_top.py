"""Top stall sites of an ncu source-page csv (SASS), plus totals per warp-role region."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src = hdr.index("Source")
i_ex = hdr.index("Instructions Executed")
tot = sum(float(r[i_s] or 0) for r in data)
print("total samples", tot)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for k, r in sorted(enumerate(data), key=lambda kr: -float(kr[1][i_s] or 0))[:n]:
    print(f"{float(r[i_s]) / tot * 100:5.1f}% line{k:5d} {r[i_src][:90]} ex={r[i_ex]}")
