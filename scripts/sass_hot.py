"""Summarise an ncu source page (--page source --csv --print-source sass):
top SASS instructions by stall samples with their dominant stall reasons, and
the stall-reason totals. python scripts/sass_hot.py page.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {s: 0.0 for s in stalls}
recs = []
for r in data:
    if len(r) != len(hdr):
        continue
    try:
        smp = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    st = {s: float(r[ix[s]] or 0) for s in stalls}
    for s in stalls:
        tot[s] += st[s]
    recs.append((smp, r[ix["Address"]], r[ix["Source"]], r[ix["Instructions Executed"]], st))
all_s = sum(x[0] for x in recs)
print("total samples", all_s)
print("stalls:", ", ".join("%s %.1f%%" % (k[6:], 100 * v / max(all_s, 1)) for k, v in
                          sorted(tot.items(), key=lambda kv: -kv[1])[:8]))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for smp, a, src, ex, st in sorted(recs, key=lambda x: -x[0])[:N]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:2]
    print("%5.1f%% %6s %-60s exec %-8s %s" % (100 * smp / max(all_s, 1), a, src[:60], ex,
                                            " ".join("%s:%d" % (k[6:], v) for k, v in top if v)))
