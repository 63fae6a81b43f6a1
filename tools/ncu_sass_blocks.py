"""Per-SASS-instruction execution counts from `ncu -i rep --page source --csv --print-source sass`:
total, and the hottest straight-line stretches (instructions with equal execution counts
grouped), to find where warp-instructions go when source attribution is ambiguous.
usage: ncu_sass_blocks.py sass.csv [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
hdr = None
ins = []
for r in rows:
    if r and r[0] == "Address":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None or not r or not r[0].startswith("0x"):
        continue
    e = r[hdr["Instructions Executed"]]
    t = r[hdr["Thread Instructions Executed"]]
    ins.append((int(r[0], 16), r[1].strip(), int(e) if e.isdigit() else 0, int(t) if t.isdigit() else 0))
tot = sum(x[2] for x in ins)
print(f"total warp-instr {tot/1e6:.1f}M over {len(ins)} SASS instructions")
# group consecutive instructions with the same execution count
blocks = []
cur = None
for k, (a, s, e, t) in enumerate(ins):
    if cur and e == cur[2] and e > 0:
        cur[1] = k
        cur[3] += e
    else:
        cur = [k, k, e, e]
        blocks.append(cur)
blocks.sort(key=lambda b: -b[3])
base = ins[0][0]
for b0, b1, e, s in blocks[:n]:
    print(f"{s/1e6:7.1f}M  {b1-b0+1:4d} instr x {e/1e3:8.1f}K  @{ins[b0][0]-base:#07x}..{ins[b1][0]-base:#07x}  "
          f"lanes {ins[b0][3]/max(1,e):4.1f}  {ins[b0][1][:50]}")
