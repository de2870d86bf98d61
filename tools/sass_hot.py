"""Summarise an ncu SASS source page: stall samples by opcode and the hottest
instructions.  usage: ncu -i rep --page source --csv --launch-skip K
--launch-count 1 --print-source sass > f.csv; python tools/sass_hot.py f.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
print(rows[0][1][:100])
hdr = rows[1]
si = hdr.index("Source")
wi = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[wi] or 0), int(r[ie] or 0), r[0], r[si].strip()))
    except (ValueError, IndexError):
        pass
tot = max(1, sum(d[0] for d in data))
itot = max(1, sum(d[1] for d in data))
by_op = collections.Counter()
inst_op = collections.Counter()
for s, n, a, src in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    by_op[op] += s
    inst_op[op] += n
print(f"total samples {tot}, warp-instructions {itot}")
for op, s in by_op.most_common(14):
    print(f"  {op:10s} stall {100*s/tot:5.1f}%   inst {100*inst_op[op]/itot:5.1f}%")
print("hottest:")
for s, n, a, src in sorted(data, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(f"  {100*s/tot:5.1f}% {a[-5:]} {src[:80]}")
