"""Opcode histogram (executed warp instructions, stall samples) of one
kernel from `ncu -i rep --page source --csv --print-source sass`."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
ia, ie, iss = (hdr.index(x) for x in ("Source", "Instructions Executed",
                                       "Warp Stall Sampling (All Samples)"))
data = []
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or r[0] == "Address":
        continue
    try:
        data.append((r[ia].strip(), int(r[ie] or 0), int(r[iss] or 0)))
    except ValueError:
        continue
te = sum(d[1] for d in data)
ts = sum(d[2] for d in data)
print("total warp instructions", te, "stall samples", ts)
c, cs = Counter(), Counter()
for src, e, s in data:
    t = src.split()
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    c[op] += e
    cs[op] += s
for op, e in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{op:12s} {e / te * 100:5.1f}% instr  {cs[op] / max(ts, 1) * 100:5.1f}% stall samples")
if len(sys.argv) > 3:  # top stall lines
    for src, e, s in sorted(data, key=lambda d: -d[2])[: int(sys.argv[3])]:
        print(f"{s:7d} {e:9d}  {src}")
