"""Summarise an ncu --page source --print-source sass CSV: hottest SASS lines and totals."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
ie = lambda d: int(d["Instructions Executed"] or 0)
st = lambda d: int(d["Warp Stall Sampling (All Samples)"] or 0)
tot_i = sum(ie(d) for d in data)
tot_s = sum(st(d) for d in data)
print(f"total warp instr {tot_i:,}  stall samples {tot_s:,}")
# group by opcode
from collections import Counter
op_i, op_s = Counter(), Counter()
for d in data:
    src = d["Source"].strip()
    parts = src.split()
    op = parts[0] if not parts[0].startswith("@") else parts[1]
    op = op.split(".")[0]
    op_i[op] += ie(d)
    op_s[op] += st(d)
print("by opcode (instr %, stall %):")
for op, v in op_i.most_common(25):
    print(f"  {op:10s} {100*v/tot_i:6.2f}%  {100*op_s[op]/max(tot_s,1):6.2f}%")
print("hottest lines by stall samples:")
for i, d in enumerate(sorted(range(len(data)), key=lambda k: -st(data[k]))[:top]):
    dd = data[d]
    print(f"{d:5d} {st(dd):7d} {ie(dd):12,d} {dd['Source'].strip()[:80]}")
