"""GPU probe: what sets the config-4 step time. Evaluates the bench's
config-4 batch with per-test records, splits the variants by the status of
their first test (completed / trap / budget) and times each class alone as
its own resident batch; prints one JSON line per class."""
import gzip
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
with gzip.open(os.path.join(ROOT, "bench_data", "cand_conv-bn_s1.txt.gz"), "rt") as f:
    cands = [x for x in f.read().splitlines() if x.strip()][:n]
ir, gen = gevo.authored_kernel("conv-bn")
suite = gevo.Suite.from_spec(ir, gen, 3, gevo.train_seed(1))
cfg = suite.exec_config()
b = suite.batch()
for c in cands:
    b.add_patch(c)
gevo.spin_counters(reset=True)
v, t, st = b.eval(cfg, tolerance=0.01, early_exit=True, tests=True)
print(json.dumps({"all": len(cands), "ms": st.device_ms, "spins": gevo.spin_counters(reset=True)}))
s0 = t["status"][:, 0]
for name, cls in (("completed", 0), ("trap", 1), ("budget", 2)):
    idx = np.nonzero(s0 == cls)[0]
    if len(idx) == 0:
        continue
    bb = suite.batch()
    for i in idx:
        bb.add_patch(cands[i])
    bb.make_resident()
    bb.eval_resident(cfg, tolerance=0.01, early_exit=True)
    _, st2 = bb.eval_resident(cfg, tolerance=0.01, early_exit=True)
    irs = t["ir"][idx, 0]
    print(json.dumps({"class": name, "variants": int(len(idx)), "ms": st2.device_ms,
                      "ir_test0_mean": float(irs.mean()), "ir_test0_max": int(irs.max()),
                      "jumps": int(t["pad"][idx, 0, 0].sum()) if t["pad"].ndim == 3 else None}))
# slowest single variants of the budget class, alone
idx = np.nonzero(s0 == 2)[0][:8]
for i in idx:
    bb = suite.batch().add_patch(cands[i])
    _, _, st3 = bb.eval(cfg, tolerance=0.01, early_exit=True)
    print(json.dumps({"budget_variant": int(i), "ms": st3.device_ms, "ir": int(t["ir"][i, 0]),
                      "cost": int(t["cost"][i, 0]), "patch": cands[i][:300]}))
