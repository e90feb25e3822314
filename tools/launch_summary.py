"""Summarise an ncu --csv launch list: per kernel count, mean time, share, DRAM MB.
python tools/launch_summary.py launches.csv"""
import csv, sys
from collections import OrderedDict
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = OrderedDict()
for r in rows:
    if "Kernel Name" in r and "Metric Name" in r:
        hdr = r; continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    k = d["Kernel Name"][:70]; m = d["Metric Name"]
    try:
        v = float(d["Metric Value"].replace(",", ""))
    except ValueError:
        continue
    a = agg.setdefault(k, {})
    a.setdefault(m, []).append(v)
tot = sum(sum(a.get("gpu__time_duration.sum", [0])) for a in agg.values())
out = []
for k, a in agg.items():
    t = a.get("gpu__time_duration.sum", [0])
    unit_scale = 1.0
    rd = sum(a.get("dram__bytes_read.sum", [0])) / max(1, len(t))
    wr = sum(a.get("dram__bytes_write.sum", [0])) / max(1, len(t))
    out.append((sum(t), len(t), sum(t) / len(t), rd, wr, k))
for s, n, m, rd, wr, k in sorted(out, reverse=True):
    print(f"{n:3d} x {m:10.1f}  share {100*s/tot:5.1f}%  dram rd {rd:10.3g} wr {wr:10.3g}  {k}")
