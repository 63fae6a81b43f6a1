"""Per-kernel table of an `ncu --metrics ... --csv` run (stdout captured to a file that may
also hold other lines): one row per launch, one column per metric.
usage: python tools/ncu_metrics_table.py file.csv"""
import csv
import sys

lines = open(sys.argv[1], errors="replace").read().splitlines()
start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
h = rows[0]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
launches, metrics = {}, []
for r in rows[1:]:
    if len(r) <= vi:
        continue
    key = (int(r[ii]), r[ki].split("(")[0].replace("void ", "").replace("dpd::", ""))
    launches.setdefault(key, {})[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    if r[mi] not in metrics:
        metrics.append(r[mi])
print("| launch | kernel | " + " | ".join(metrics) + " |")
print("|---|---|" + "---|" * len(metrics))
for (i, k), m in sorted(launches.items()):
    print(f"| {i} | {k[:40]} | " + " | ".join(m.get(x, "") for x in metrics) + " |")
