"""Warp-instruction, lane and shared-wavefront totals per source region of an ncu source-page
CSV (`ncu -i rep --page source --csv --print-source cuda,sass`).  A region of the tile kernel
file is the nearest enclosing function header or `// ----` phase comment above the line.
usage: ncu_regions.py src.csv kernel_file.cuh [n]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
kfile = sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
src = open(kfile).read().split("\n")
kname = kfile.split("/")[-1]


def region(line):
    for k in range(line - 1, -1, -1):
        t = src[k]
        if t.startswith(("__device__", "template", "__global__")) or "// ----" in t:
            return t.strip()[:64]
    return "?"


def num(x):
    return int(x) if x.lstrip("-").isdigit() else 0


agg = collections.defaultdict(collections.Counter)
fname = hdr = None
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
    key = region(int(r[0])) if fname == kname else fname
    c = agg[key]
    c["ins"] += num(r[hdr["Instructions Executed"]])
    c["tin"] += num(r[hdr["Thread Instructions Executed"]])
    c["wf"] += num(r[hdr["L1 Wavefronts Shared"]])
    c["samp"] += num(r[hdr["Warp Stall Sampling (All Samples)"]])
    for k, i in hdr.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            c[k] += num(r[i])
ti = sum(c["ins"] for c in agg.values())
tw = sum(c["wf"] for c in agg.values())
ts = sum(c["samp"] for c in agg.values())
print(f"total warp-instr {ti/1e6:.1f}M  smem wavefronts {tw/1e6:.1f}M")
for k, c in sorted(agg.items(), key=lambda kv: -kv[1]["ins"])[:n]:
    st = sorted(((v, s[6:]) for s, v in c.items() if s.startswith("stall_")), reverse=True)[:3]
    print(f"{c['ins']/1e6:7.1f}M {100*c['ins']/ti:5.1f}%  lanes {c['tin']/max(1,c['ins']):4.1f}  "
          f"wf {c['wf']/1e6:6.1f}M  samples {100*c['samp']/max(1,ts):5.1f}% "
          f"({' '.join(f'{n}:{100*v/max(1,c[chr(115)+chr(97)+chr(109)+chr(112)]):.0f}%' for v, n in st)})  {k}")
