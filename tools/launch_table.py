"""Tables from an ncu --csv launch list (--metrics ...):
  python tools/launch_table.py agg  FILE.csv   per kernel: launches, mean us, total ms, share of device time
  python tools/launch_table.py each FILE.csv   per launch: us, DRAM read/write MB and any other metric"""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(.*$", "", name) if not name.startswith("void cub") else name[:60]
    name = name.replace("qmcg::", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    return name[:60]


def rows(path):
    hdr, out = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            key = int(d["ID"])
            e = out.setdefault(key, {"name": short(d["Kernel Name"])})
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return list(out.values())


mode, path = sys.argv[1], sys.argv[2]
launches = rows(path)
if mode == "agg":
    agg = collections.OrderedDict()
    for e in launches:
        a = agg.setdefault(e["name"], [0, 0.0])
        a[0] += 1
        a[1] += e["gpu__time_duration.sum"] / 1e3
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':60s} {'launches':>9s} {'mean us':>10s} {'total ms':>10s} {'share':>7s}")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:60s} {n:9d} {us / n:10.2f} {us / 1e3:10.2f} {100 * us / tot:6.2f}%")
else:
    extra = [k for k in launches[0] if k not in ("name", "gpu__time_duration.sum", "dram__bytes_read.sum",
                                                    "dram__bytes_write.sum")]
    print(f"{'id':>3s} {'kernel':46s} {'us':>9s} {'DRAM rd MB':>11s} {'DRAM wr MB':>11s} " +
          " ".join(f"{k.split('.')[0][-14:]:>14s}" for k in extra))
    for i, e in enumerate(launches):
        print(f"{i:3d} {e['name'][:46]:46s} {e['gpu__time_duration.sum'] / 1e3:9.1f} "
              f"{e.get('dram__bytes_read.sum', 0) / 1e6:11.1f} {e.get('dram__bytes_write.sum', 0) / 1e6:11.1f} " +
              " ".join(f"{e.get(k, 0):14.1f}" for k in extra))
