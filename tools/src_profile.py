"""Summarise an `ncu -i REP --page source --csv --print-source sass` dump: dynamic instruction mix
(warp-level executions per opcode) and the stall samples per opcode and per reason (profiling aid)."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Source" in r)
hdr = rows[hdr_i]
data = rows[hdr_i + 1:]
ci = {h: i for i, h in enumerate(hdr)}
ex = collections.Counter()
st = collections.Counter()
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
rs = collections.Counter()
tot_ex = 0
for r in data:
    if len(r) < len(hdr):
        continue
    src = r[ci["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    n = int(r[ci["Instructions Executed"]] or 0)
    ex[op] += n
    tot_ex += n
    st[op] += int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    for h in reasons:
        rs[h] += int(r[ci[h]] or 0)
print(f"total warp instructions executed: {tot_ex}")
for op, n in ex.most_common(25):
    print(f"  {op:10s} {n:10d} {100.0 * n / tot_ex:5.1f}%   stall samples {st[op]}")
tot_s = sum(rs.values())
print("stall samples by reason:")
for h, n in rs.most_common(12):
    print(f"  {h:28s} {n:8d} {100.0 * n / max(tot_s, 1):5.1f}%")
