"""Phase breakdown of a kernel from `ncu --page source --csv --print-source cuda,sass`.
usage: ncu_phases.py file.csv phases.txt
phases.txt lines: `<file-substring> <lo>-<hi> <label>`; unmatched lines go to `other:<file>`.
Prints per phase: warp-instr share, lane efficiency, stall-sample share, top stall reasons."""
import collections
import csv
import sys


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


rows = list(csv.reader(open(sys.argv[1], errors="replace")))
spec = []
for ln in open(sys.argv[2]):
    ln = ln.split("#")[0].split()
    if len(ln) == 3:
        lo, hi = ln[1].split("-")
        spec.append((ln[0], int(lo), int(hi), ln[2]))
agg = collections.defaultdict(lambda: collections.Counter())
hdr = None
fname = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r) if k not in hdr_dupe} if False else None
        hdr = {}
        for i, k in enumerate(r):
            hdr.setdefault(k, i)
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    line = int(r[0])
    lab = None
    for f, lo, hi, name in spec:
        if f in fname and lo <= line <= hi:
            lab = name
            break
    if lab is None:
        lab = "other:" + fname.split("/")[-1]
    c = agg[lab]
    c["inst"] += num(r[hdr["Instructions Executed"]])
    c["tinst"] += num(r[hdr["Thread Instructions Executed"]])
    c["samp"] += num(r[hdr["Warp Stall Sampling (All Samples)"]])
    c["wf"] += num(r[hdr["L1 Wavefronts Shared"]])
    c["wfi"] += num(r[hdr["L1 Wavefronts Shared Ideal"]])
    for k, i in hdr.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            c[k] += num(r[i])
ti = sum(c["inst"] for c in agg.values())
ts = sum(c["samp"] for c in agg.values())
tw = sum(c["wf"] for c in agg.values())
print(f"total warp-instr {ti:,}  samples {ts:,}  smem wavefronts {tw:,}")
for lab, c in sorted(agg.items(), key=lambda kv: -kv[1]["inst"]):
    st = sorted(((v, k[6:]) for k, v in c.items() if k.startswith("stall_")), reverse=True)[:4]
    eff = c["tinst"] / max(1, c["inst"]) / 32
    print(f"{lab:24s} instr {100*c['inst']/ti:5.1f}%  lanes {100*eff:4.0f}%  samples {100*c['samp']/max(1,ts):5.1f}%  "
          f"samp/instr(norm) {c['samp']/max(1,ts)/(c['inst']/ti+1e-12):4.2f}  "
          f"smem-wf {100*c['wf']/max(1,tw):4.1f}% (ideal {100*c['wfi']/max(1,tw):4.1f}%)  " +
          " ".join(f"{k}:{100*v/max(1,c['samp']):.0f}%" for v, k in st))
