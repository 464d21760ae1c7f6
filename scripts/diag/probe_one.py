"""Times single candidates (bench sample, seed 1) with both interpreters:
python scripts/probe_one.py bench:idx [bench:idx ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

for arg in sys.argv[1:]:
    bench, idx = arg.split(":")
    idx = int(idx)
    cand = gevo.sample_candidates(bench, 1024, 1, 4)[idx]
    for ntests in (16, 1):
        suite = gevo.Suite.from_benchmark(bench, ntests, gevo.train_seed(1))
        cfg = suite.exec_config()
        b = suite.batch().add_patch(cand)
        for seq in (False, True):
            ms = []
            for _ in range(4):
                gevo.tp_counters(reset=True)
                v, t, st = b.eval(cfg, early_exit=True, tests=True, sequential=seq)
                ms.append(round(st.device_ms, 4))
            r = t[0, 0]
            print(bench, idx, "tests", ntests, "seq" if seq else "tp", ms, "status", int(r["status"]),
                  "ir", int(r["ir"]), "jumps", int(r["pad"][0]), "rerun", gevo.tp_counters()[0],
                  flush=True)
