"""Per-source-line summary of an ncu report (--import-source on, -lineinfo):
  ncu -i r.ncu-rep --page source --csv --print-source cuda,sass > r.csv
  python scripts/ncu_lines.py r.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = []
for r in rows[3:]:
    if len(r) > 8 and r[2] == "-":
        try:
            out.append((float(r[4]), float(r[7]), r[0], r[1][:90]))
        except ValueError:
            pass
ts = sum(x[0] for x in out) or 1
ti = sum(x[1] for x in out) or 1
print("samples %d  instructions %d" % (ts, ti))
for s, i, line, src in sorted(out, reverse=True)[:top]:
    print("%5.1f%% samples %5.1f%% inst  L%-5s %s" % (100 * s / ts, 100 * i / ti, line, src.strip()))
