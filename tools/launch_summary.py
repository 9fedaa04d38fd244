"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"].split("(")[0]
            unit = d.get("Metric Unit", "ns")
            v = float(d["Metric Value"].replace(",", "")) * (1e3 if unit == "us" else (1e6 if unit == "ms" else 1))
            c, t = agg.get(k, (0, 0.0))
            agg[k] = (c + 1, t + v)
tot = sum(t for _, t in agg.values())
print("| kernel | launches | total ms | share |\n|---|---|---|---|")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| {k} | {c} | {t / 1e6:.3f} | {t / tot:.1%} |")
