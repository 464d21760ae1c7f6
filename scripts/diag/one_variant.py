"""Evaluate one bench candidate alone (all tests) a few times -- an ncu target:
  ncu ... -k regex:interp_tp -s 1 -c 1 python scripts/one_variant.py nw-sync 721"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

bench, idx = sys.argv[1], int(sys.argv[2])
cands = gevo.sample_candidates(bench, 1024, 1, 4)
suite = gevo.Suite.from_benchmark(bench, 16, gevo.train_seed(1))
cfg = suite.exec_config()
b = suite.batch()
b.add_patch(cands[idx])
for _ in range(3):
    _, _, st = b.eval(cfg, early_exit=True)
    print(bench, idx, "%.4f ms" % st.device_ms)
