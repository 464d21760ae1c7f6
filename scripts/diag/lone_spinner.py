"""Runs one spinning variant (candidate index from sample_candidates) on one
test, for per-IR latency profiling: python scripts/lone_spinner.py <bench> <idx>"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

bench, idx = sys.argv[1], int(sys.argv[2])
cand = gevo.sample_candidates(bench, idx + 1, 1, 4)[idx]
s1 = gevo.Suite.from_benchmark(bench, 1, gevo.train_seed(1))
b1 = s1.batch().add_patch(cand)
b1.make_resident()
vr, st = b1.eval_resident(s1.exec_config(), records=True)
print(bench, idx, "ms", st.device_ms, "ir", int(vr["ir_ref"][0]),
      "cycles/IR", st.device_ms * 1.965e6 / max(int(vr["ir_ref"][0]), 1))
