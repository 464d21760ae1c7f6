"""GPU probe: dump chosen bench candidates (IR, per-test records, device ms on
the thread-parallel and sequential-lane interpreters).
  python scripts/probe_var.py nw-sync 356 721 ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

bench, idx = sys.argv[1], [int(x) for x in sys.argv[2:]]
cands = gevo.sample_candidates(bench, 1024, 1, 4)
suite = gevo.Suite.from_benchmark(bench, 16, gevo.train_seed(1))
cfg = suite.exec_config()
for i in idx:
    b = suite.batch()
    b.add_patch(cands[i])
    b.eval(cfg, early_exit=True)
    gevo.tp_counters(reset=True)
    _, tr, st = b.eval(cfg, early_exit=True, tests=True)
    rr = gevo.tp_counters(reset=True)[0]
    _, _, sq = b.eval(cfg, early_exit=True, sequential=True)
    ir, _ = gevo.apply_patch(gevo.benchmark_ir(bench), cands[i])
    print("# variant %d  tp %.3f ms  seq %.3f ms  reruns %d" % (i, st.device_ms, sq.device_ms, rr))
    print("# patch", cands[i])
    for k in range(tr.shape[1]):
        r = tr[0, k]
        print("#  test %d status %d code %d ir %d cost %d jumps %d" %
              (k, r["status"], r["code"], r["ir"], r["cost"], r["pad"][0]))
    print(ir)
