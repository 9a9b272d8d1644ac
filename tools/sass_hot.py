"""Top SASS instructions by warp-stall samples from an `ncu --page source --print-source sass --csv` dump."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)")
ii = hdr.index("Instructions Executed")
data = [r for r in rows[2:] if len(r) > si]
tot = sum(float(r[si] or 0) for r in data)
print(f"total samples {tot:.0f}, instructions {len(data)}")
top = sorted(data, key=lambda r: -float(r[si] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for r in top:
    print(f"{float(r[si]):7.0f} {100 * float(r[si]) / tot:5.1f}%  exec {r[ii]:>8}  {r[0][-5:]}  {r[1].strip()[:80]}")
