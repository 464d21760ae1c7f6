"""Per-launch issue counts of the interpreter for bench.py's roofline.

Run on the GPU box:
  ncu --metrics smsp__inst_executed.sum,smsp__thread_inst_executed.sum,gpu__time_duration.sum,\
dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:interp --csv \
      --log-file gpurun_out/issue.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline
  python scripts/issue_profile.py gpurun_out/issue.csv profiles/issue_per_launch.json

bench.py evaluates the workload kernels in a fixed order (hot-branch, nw-sync,
bfs-load) in every pass, so launch i belongs to KERNELS[i % 3]. Counts are the
median over the passes (the thread-parallel kernel's aborts make them vary a
little between runs)."""
import csv
import json
import statistics
import sys

KERNELS = ("hot-branch", "nw-sync", "bfs-load")

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
per = {}
for r in rows[hdr + 1:]:
    d = dict(zip(h, r))
    per.setdefault(int(d["ID"]), {"name": d["Kernel Name"]})[d["Metric Name"]] = (
        float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
launches = [per[k] for k in sorted(per) if "interp" in per[k]["name"]]
out = {"kernels": {}, "source": sys.argv[1]}
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for i, k in enumerate(KERNELS):
    mine = launches[i::3]
    if not mine:
        continue

    def med(metric, conv):
        xs = [m[metric][0] * conv(m[metric][1]) for m in mine if metric in m]
        return statistics.median(xs) if xs else None

    out["kernels"][k] = {
        "launches": len(mine),
        "warp_inst": med("smsp__inst_executed.sum", lambda u: 1),
        "thread_inst": med("smsp__thread_inst_executed.sum", lambda u: 1),
        "ncu_ms": med("gpu__time_duration.sum", lambda u: scale.get(u, 1)),
        "dram_bytes": (med("dram__bytes_read.sum", lambda u: bscale.get(u, 1)) or 0) +
                      (med("dram__bytes_write.sum", lambda u: bscale.get(u, 1)) or 0),
        "kernel": mine[0]["name"].split("(")[0],
    }
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
