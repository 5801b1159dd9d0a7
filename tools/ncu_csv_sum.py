"""Summarise an ncu --csv launch list: per kernel name, launches and mean of each metric."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = (d["Kernel Name"][:70], d["Metric Name"])
        v = float(d["Metric Value"].replace(",", ""))
        agg.setdefault(k, []).append(v)
for (name, met), vs in agg.items():
    print(f"{name:70s} {met:28s} n={len(vs):4d} mean={sum(vs) / len(vs):.4g}")
