"""Evaluate one bench batch (default: nw-sync, 1024 mutants x 16 tests) a few
times -- a target for ncu captures of a single interpreter launch:
  ncu ... -k regex:interp_tp -s 1 -c 1 python scripts/one_batch.py nw-sync"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

bench = sys.argv[1] if len(sys.argv) > 1 else "nw-sync"
pop = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
cands = gevo.sample_candidates(bench, pop, 1, 4)
suite = gevo.Suite.from_benchmark(bench, 16, gevo.train_seed(1))
cfg = suite.exec_config()
b = suite.batch()
for c in cands:
    b.add_patch(c)
b.make_resident()
for _ in range(3):
    _, st = b.eval_resident(cfg, early_exit=True)
    print(bench, "%.4f ms" % st.device_ms)
