"""Issue counts of one bench step of a workload, for bench.py's roofline.

Run on the GPU box (bench.py --profile-step brackets exactly one untimed step
of the workload with cudaProfilerStart/Stop):
  ncu --profile-from-start off --metrics smsp__inst_executed.sum,\
smsp__thread_inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,\
dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/issue_c4.csv \
      python bench.py --profile-step config4
  python scripts/issue_profile.py config4 gpurun_out/issue_c4.csv profiles/issue_per_launch.json

Sums every interpreter launch of the step (a batch larger than the scratch
budget runs in several launches) and lists the other kernels beside them.
The output file keeps one entry per workload."""
import csv
import json
import os
import sys

workload, src, dst = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(src)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
per = {}
for r in rows[hdr + 1:]:
    d = dict(zip(h, r))
    per.setdefault(int(d["ID"]), {"name": d["Kernel Name"]})[d["Metric Name"]] = (
        float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def val(m, metric, conv):
    return m[metric][0] * conv(m[metric][1]) if metric in m else 0.0


interp = [per[k] for k in sorted(per) if "interp" in per[k]["name"]]
others = [per[k] for k in sorted(per) if "interp" not in per[k]["name"]]
entry = {
    "launches": len(interp),
    "kernel": interp[0]["name"].split("(")[0] if interp else None,
    "warp_inst": sum(val(m, "smsp__inst_executed.sum", lambda u: 1) for m in interp),
    "thread_inst": sum(val(m, "smsp__thread_inst_executed.sum", lambda u: 1) for m in interp),
    "ncu_ms": sum(val(m, "gpu__time_duration.sum", lambda u: scale.get(u, 1)) for m in interp),
    "dram_bytes": sum(val(m, "dram__bytes_read.sum", lambda u: bscale.get(u, 1)) +
                      val(m, "dram__bytes_write.sum", lambda u: bscale.get(u, 1)) for m in interp),
    "other_kernels": [{"kernel": m["name"].split("(")[0],
                       "ncu_ms": val(m, "gpu__time_duration.sum", lambda u: scale.get(u, 1))}
                      for m in others],
    "source": src,
}
out = json.load(open(dst)) if os.path.exists(dst) else {}
out.setdefault("workloads", {})[workload] = entry
out.pop("kernels", None)
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(entry, indent=1))
