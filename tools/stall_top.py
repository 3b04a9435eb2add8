"""Per-reason top SASS lines from an `ncu --page source --csv --print-source sass` dump (profiling aid)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0] if "Source" in rows[0] else rows[1]
data = rows[1:] if hdr is rows[0] else rows[2:]
src = hdr.index("Source")
n = int(sys.argv[3]) if len(sys.argv) > 3 else 6
for reason in sys.argv[2].split(","):
    c = hdr.index(reason)
    tot = sum(int(r[c] or 0) for r in data)
    print(f"== {reason}: {tot}")
    for i, r in sorted(enumerate(data), key=lambda x: -int(x[1][c] or 0))[:n]:
        print(f"  {int(r[c] or 0):6d} @{i:5d} {r[src][:90]}")
