"""GPU probe: the slowest CTAs of a corpus-kernel candidate batch (per-CTA
clock), with their variants' records and patches.
Usage: slow_variants.py <kernel> <pop> <tests> [top]"""
import json
import os
import sys

os.environ.setdefault("GEVO_CTA_CLOCK", "1")
import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

k, P, T = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 8
cands = gevo.sample_candidates(k, P, 1, 4)
suite = gevo.Suite.from_benchmark(k, T, gevo.train_seed(1))
cfg = suite.exec_config()
b = suite.batch()
for c in cands:
    b.add_patch(c)
gevo.tp_counters(reset=True)
v, t, st = b.eval(cfg, early_exit=True, tests=True)
clk = gevo.debug_cta_clock(P, T).astype(np.int64)
ran = clk[:, :, 0] > 0
dur = (clk[:, :, 1] - clk[:, :, 0]) / 1e6
print(json.dumps({"kernel": k, "pop": P, "tests": T, "device_ms": st.device_ms,
                  "launches": st.launches, "tp": gevo.tp_counters(reset=True)}))
order = np.argsort(-dur, axis=None)[:top]
for kk in order:
    vi, ti = divmod(int(kk), T)
    if not ran[vi, ti]:
        continue
    print(json.dumps({"variant": vi, "test": ti, "ms": float(dur[vi, ti]),
                      "status": int(t["status"][vi, ti]), "code": int(t["code"][vi, ti]),
                      "ir": int(t["ir"][vi, ti]), "jumps": int(t["pad"][vi, ti, 0]),
                      "patch": cands[vi]}))
