"""GPU probe: full bench batches (1024 mutants x 16 tests per kernel) -- device
ms of the thread-parallel and sequential interpreters, re-run counts, and the
batch time with the k slowest variants (timed alone) removed, to separate tail
from throughput."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2004_08140_b200 as gevo  # noqa: E402

BENCHES = sys.argv[1:] or ["hot-branch", "nw-sync", "bfs-load"]


def timed(suite, cfg, cands, **kw):
    b = suite.batch()
    for c in cands:
        b.add_patch(c)
    b.make_resident()
    b.eval_resident(cfg, early_exit=True)
    gevo.tp_counters(reset=True)
    ms = []
    for _ in range(3):
        _, st = b.eval_resident(cfg, early_exit=True)
        ms.append(st.device_ms)
    return min(ms), gevo.tp_counters(reset=True)


for bench in BENCHES:
    cands = gevo.sample_candidates(bench, 1024, 1, 4)
    suite = gevo.Suite.from_benchmark(bench, 16, gevo.train_seed(1))
    cfg = suite.exec_config()
    full, cnt = timed(suite, cfg, cands)
    solo = []
    for i, c in enumerate(cands):
        b = suite.batch()
        b.add_patch(c)
        b.eval(cfg, early_exit=True)
        gevo.tp_counters(reset=True)
        _, _, st = b.eval(cfg, early_exit=True)
        solo.append((st.device_ms, i, gevo.tp_counters(reset=True)[0]))
    solo.sort(reverse=True)
    out = {"bench": bench, "full_ms": full, "reruns_per_eval": cnt[0] / 3, "tp_instances": cnt[1] / 3,
           "top": [(round(t, 3), i, r) for t, i, r in solo[:12]],
           "solo_median": solo[len(solo) // 2][0],
           "variants_with_reruns": sum(1 for s in solo if s[2])}
    for k in (1, 4, 16, 64):
        drop = {i for _, i, _ in solo[:k]}
        out["drop%d_ms" % k] = timed(suite, cfg, [c for i, c in enumerate(cands) if i not in drop])[0]
    rr = {i for _, i, r in solo if r}
    out["drop_rerun_ms"] = timed(suite, cfg, [c for i, c in enumerate(cands) if i not in rr])[0]
    print(json.dumps(out), flush=True)
