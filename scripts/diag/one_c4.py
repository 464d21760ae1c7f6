"""GPU probe: one config-4 candidate alone (batch of one), its IR, records and
CTA times. Usage: [C4_SEED=s] one_c4.py <candidate index> [...]"""
import gzip
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ.setdefault("GEVO_CTA_CLOCK", "1")
import paper_2004_08140_b200 as gevo  # noqa: E402

SEED = int(os.environ.get("C4_SEED", "1"))  # committed candidate set
with gzip.open(os.path.join(ROOT, "bench_data", "cand_conv-bn_s%d.txt.gz" % SEED), "rt") as f:
    cands = [x for x in f.read().splitlines() if x.strip()]
ir, gen = gevo.authored_kernel("conv-bn")
suite = gevo.Suite.from_spec(ir, gen, 3, gevo.train_seed(1))
cfg = suite.exec_config()
for a in sys.argv[1:]:
    i = int(a)
    text, _ = gevo.apply_patch(ir, cands[i])
    print("==== candidate", i, cands[i])
    print(text)
    b = suite.batch().add_patch(cands[i])
    gevo.spin_counters(reset=True)
    gevo.work_counters(reset=True)
    _, t, st = b.eval(cfg, tolerance=0.01, early_exit=False, tests=True)
    print(json.dumps({"spins": gevo.spin_counters(reset=True), "interpreted": gevo.work_counters(reset=True)}))
    clk = gevo.debug_cta_clock(1, 3)
    for tt in range(3):
        r = t[0, tt]
        print(json.dumps({"test": tt, "status": int(r["status"]), "code": int(r["code"]),
                          "ir": int(r["ir"]), "ms": (int(clk[0, tt, 1]) - int(clk[0, tt, 0])) / 1e6}))
    print("device_ms", st.device_ms)
