"""Text summary of one ncu --set full capture (the profiles/r2_ncu_full_*.txt
format): details page, warp stall reasons per issued instruction, a few raw
counters, and SASS opcode classes by stall samples / executed instructions.

  python scripts/ncu_summary.py report.ncu-rep "<header line>" ["<command line>"] > out.txt"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def page(*args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], check=True, capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


print("# " + (sys.argv[2] if len(sys.argv) > 2 else rep))
if len(sys.argv) > 3:
    print("# command: " + sys.argv[3])
print()
rows = page("--page", "details")
h = rows[0]
for r in rows[1:]:
    d = dict(zip(h, r))
    name = d.get("Metric Name", "")
    if name:
        print("%s | %s | %s | %s" % (d.get("Section Name", ""), name, d.get("Metric Unit", ""),
                                     d.get("Metric Value", "")))
    elif d.get("Rule Name"):
        print("%s | %s | %s" % (d.get("Rule Type", "OPT"), d.get("Rule Description", "")[:400],
                                d.get("Estimated Speedup", "")))
raw = page("--page", "raw")
hr, val = raw[0], raw[2]
d = dict(zip(hr, val))
print("\n## warp stall reasons (warps stalled per issued instruction)")
st = []
for k, v in d.items():
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            st.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
for v, k in sorted(st, reverse=True):
    print("%-40s %.3f" % (k, v))
for k in ("smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg",
          "dram__bytes_read.sum", "dram__bytes_write.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"):
    if k in d:
        print(k, d[k])
src = page("--page", "source", "--print-source", "sass")
hs = next(i for i, r in enumerate(src) if r and "Source" in r)
h = src[hs]
ci = h.index("Source")
si = next(i for i, x in enumerate(h) if x.startswith("Warp Stall Sampling (All"))
ii = next(i for i, x in enumerate(h) if x.startswith("Instructions Executed"))
samp, inst = collections.Counter(), collections.Counter()
for r in src[hs + 1:]:
    if len(r) <= max(ci, si, ii):
        continue
    op = r[ci].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else (op[1] if len(op) > 1 else op[0])
    o = o.split(".")[0]
    try:
        samp[o] += float(r[si] or 0)
        inst[o] += float(r[ii] or 0)
    except ValueError:
        pass
ts, ti = sum(samp.values()) or 1, sum(inst.values()) or 1
print("\n## SASS opcode classes: share of stall samples / of executed warp instructions")
for o, s in samp.most_common(16):
    print("%-9s %5.1f%% samples %5.1f%% inst" % (o, 100 * s / ts, 100 * inst[o] / ti))
