"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count,
mean duration and share of the total (cold-cache, serialised: compare SHARES)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for r in rows[hi + 1:]:
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("void ", "")
    v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1e-3)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':40s} {'launches':>8s} {'mean_us':>9s} {'total_us':>10s} {'share':>6s}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:40]:40s} {n:8d} {t / n:9.1f} {t:10.1f} {100 * t / tot:5.1f}%")
