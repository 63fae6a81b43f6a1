"""Top source lines of an ncu source-page CSV by shared-memory wavefronts, with warp-instr,
lane efficiency and wavefronts per instruction.  usage: ncu_lines_wf.py src.csv [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
fname = hdr = None
out = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {}
        for i, k in enumerate(r):
            hdr.setdefault(k, i)
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    g = lambda k: int(r[hdr[k]]) if r[hdr[k]].lstrip("-").isdigit() else 0
    wf, ins, tin = g("L1 Wavefronts Shared"), g("Instructions Executed"), g("Thread Instructions Executed")
    if wf or ins:
        out.append((wf, ins, tin, g("L1 Wavefronts Shared Ideal"), fname, r[0], r[1].strip()[:70]))
tw = sum(o[0] for o in out)
ti = sum(o[1] for o in out)
key = 1 if len(sys.argv) > 3 and sys.argv[3] == "instr" else 0
print(f"total wf {tw:,}  warp-instr {ti:,}")
for wf, ins, tin, wfi, f, ln, src in sorted(out, key=lambda o: -o[key])[:n]:
    print(f"{f[:14]:14s}:{ln:>4s} wf {wf/1e6:6.2f}M ideal {wfi/1e6:6.2f}M instr {ins/1e6:6.2f}M lanes {tin/max(1,ins):4.1f}  {src}")
