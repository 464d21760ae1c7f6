"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
agg = collections.OrderedDict()
for r in rows[hdr + 1:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"].split("(")[0][:60]
    v = float(d["Metric Value"].replace(",", ""))
    unit = d["Metric Unit"]
    ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
    a = agg.setdefault(name, [0, 0.0, []])
    a[0] += 1
    a[1] += ns
    a[2].append(ns)
tot = sum(a[1] for a in agg.values())
for k, (n, ns, xs) in agg.items():
    print("%-62s n=%4d total=%10.3f ms share=%5.1f%% max=%9.3f ms" % (k, n, ns / 1e6, 100 * ns / tot, max(xs) / 1e6))
