"""How much device work an in-CTA early exit could save: per bench kernel,
dynamic IR of the tests after each variant's first failing test (the
reference never runs them) against the IR of the tests up to it."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

for bench in ("hot-branch", "nw-sync", "bfs-load"):
    suite = gevo.Suite.from_benchmark(bench, 16, gevo.train_seed(1))
    cfg = suite.exec_config()
    b = suite.batch()
    for c in gevo.sample_candidates(bench, 1024, 1, 4):
        b.add_patch(c)
    vrec, tr, _ = b.eval(cfg, early_exit=False, tests=True)
    used = wasted = 0
    jumps_after = 0
    for v in range(tr.shape[0]):
        ft = int(vrec[v]["failing_test"])
        cut = tr.shape[1] if ft < 0 else ft + 1
        used += int(tr[v, :cut]["ir"].sum())
        wasted += int(tr[v, cut:]["ir"].sum())
        jumps_after += int((tr[v, cut:]["pad"][:, 0] > 0).sum()) if cut < tr.shape[1] else 0
    print(bench, "IR up to the first failure %.3g, after it %.3g (%.0f%%), spin-jumping instances after it %d" %
          (used, wasted, 100.0 * wasted / max(used + wasted, 1), jumps_after))
