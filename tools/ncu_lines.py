"""Per-source-line instruction / stall totals from `ncu --page source --csv --print-source cuda,sass`.
usage: ncu_lines.py file.csv [top] [file:lo-hi=label ...]"""
import collections
import csv
import sys


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = collections.OrderedDict()
fname = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    if r[0] != "":
        agg[(fname, int(r[0]))] = (num(r[7]), num(r[4]), r[1].strip())
tot = sum(v[0] for v in agg.values())
tots = sum(v[1] for v in agg.values())
print(f"total warp-instr {tot:,}  stall samples {tots:,}")
groups = collections.OrderedDict()
for spec in sys.argv[3:]:
    rng, label = spec.split("=")
    f, lohi = rng.split(":")
    lo, hi = map(int, lohi.split("-"))
    groups[label] = (f, lo, hi)
gs = collections.defaultdict(lambda: [0, 0])
for (f, l), (i, s, _) in agg.items():
    lab = "other:" + f
    for label, (gf, lo, hi) in groups.items():
        if f.startswith(gf) and lo <= l <= hi:
            lab = label
            break
    gs[lab][0] += i
    gs[lab][1] += s
for lab, (i, s) in sorted(gs.items(), key=lambda kv: -kv[1][0]):
    print(f"  {lab:28s} {100 * i / tot:5.1f}% instr {100 * s / tots:5.1f}% stall")
for (f, l), (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * i / tot:5.1f}% {100 * s / tots:5.1f}%st {f[:18]:18s}:{l:<4d} {src[:80]}")
