"""One evaluation of one bench candidate (for ncu): one_eval.py bench idx ntests seq(0/1) reps"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

bench, idx, nt, seq, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4] == "1", int(sys.argv[5])
cand = gevo.sample_candidates(bench, 1024, 1, 4)[idx]
suite = gevo.Suite.from_benchmark(bench, nt, gevo.train_seed(1))
b = suite.batch().add_patch(cand)
for _ in range(reps):
    v, t, st = b.eval(suite.exec_config(), early_exit=True, sequential=seq)
    print(st.device_ms)
