"""GPU probe: what sets the config-4 step time (c4_tail.py [n [seed]]). Evaluates the bench's
config-4 batch with per-test records and per-CTA timing (GEVO_CTA_CLOCK=1),
then prints: the step makespan, SM-time by the class of the variant's first
test (completed / trap / budget) and of the CTA's role (the test the reference
runs, or a speculative later test), and the longest CTAs."""
import gzip
import json
import os
import sys

os.environ.setdefault("GEVO_CTA_CLOCK", "1")
import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1  # committed candidate set
with gzip.open(os.path.join(ROOT, "bench_data", "cand_conv-bn_s%d.txt.gz" % seed), "rt") as f:
    cands = [x for x in f.read().splitlines() if x.strip()][:n]
ir, gen = gevo.authored_kernel("conv-bn")
suite = gevo.Suite.from_spec(ir, gen, 3, gevo.train_seed(1))
cfg = suite.exec_config()
b = suite.batch()
for c in cands:
    b.add_patch(c)
b.eval(cfg, tolerance=0.01, early_exit=True)
gevo.spin_counters(reset=True)
v, t, st = b.eval(cfg, tolerance=0.01, early_exit=True, tests=True)
clk = gevo.debug_cta_clock(len(cands), 3).astype(np.int64)
ran = clk[:, :, 0] > 0
t0 = clk[:, :, 0][ran].min()
dur = (clk[:, :, 1] - clk[:, :, 0]) / 1e6  # ms
end = (clk[:, :, 1] - t0) / 1e6
print(json.dumps({"variants": len(cands), "device_ms": st.device_ms, "launches": st.launches,
                  "makespan_ms": float(end[ran].max()), "ctas": int(ran.sum()),
                  "sm_ms_total": float(dur[ran].sum()), "spins": gevo.spin_counters(reset=True)}))
s0 = t["status"][:, 0]
ff = v["failing_test"]
for name, cls in (("completed", 0), ("trap", 1), ("budget", 2)):
    rows = s0 == cls
    for role in ("reference", "speculative"):
        m = np.zeros_like(ran)
        for tt in range(3):
            ref_run = (ff < 0) | (ff >= tt)
            m[:, tt] = rows & ran[:, tt] & (ref_run if role == "reference" else ~ref_run)
        if m.sum() == 0:
            continue
        print(json.dumps({"class": name, "role": role, "ctas": int(m.sum()),
                          "sm_ms": float(dur[m].sum()), "max_ms": float(dur[m].max()),
                          "mean_ms": float(dur[m].mean()),
                          "ir_mean": float(clk[:, :, 3][m].mean())}))
order = np.argsort(-dur, axis=None)[:12]
for k in order:
    vi, ti = divmod(int(k), 3)
    if not ran[vi, ti]:
        continue
    print(json.dumps({"cta": [vi, ti], "ms": float(dur[vi, ti]), "end_ms": float(end[vi, ti]),
                      "status": int(t["status"][vi, ti]), "code": int(t["code"][vi, ti]),
                      "ir": int(t["ir"][vi, ti]), "cta_ir": int(clk[vi, ti, 3]),
                      "jumps": int(t["pad"][vi, ti, 0]), "patch": cands[vi][:200]}))

# occupancy timeline (CTAs running per 50 ms) and the last CTAs to finish
ends = end[ran]
starts = (clk[:, :, 0][ran] - t0) / 1e6
span = float(ends.max())
line = []
for b in range(0, int(span) + 50, 50):
    line.append(int(((starts < b + 50) & (ends > b)).sum()))
print(json.dumps({"active_ctas_per_50ms": line}))
order = np.argsort(-end, axis=None)[:10]
for k in order:
    vi, ti = divmod(int(k), 3)
    if ran[vi, ti]:
        print(json.dumps({"late_cta": [vi, ti], "start_ms": float(end[vi, ti] - dur[vi, ti]),
                          "end_ms": float(end[vi, ti]), "status": int(t["status"][vi, ti]),
                          "ir": int(t["ir"][vi, ti])}))
