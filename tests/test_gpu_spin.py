"""Exactness of the spin accelerator (interp.cu): on spinner-rich candidate
populations (seeded validated mutants of the corpus kernels, 10^6 budget) every
per-test record -- status, reason, cycle cost, dynamic IR, error -- equals the
plain-C oracle's (oracle/evoir_oracle.c, pinned to the reference's goldens),
including the budget-exceeded runs the accelerator jumped over."""
import re

import pytest

import oracle_binding as ob
from _util import hex_double

pytestmark = pytest.mark.gpu

STATUS = {0: "completed", 1: "trap", 2: "budget"}


def _oracle_tests(gevo, bench, n, seed):
    docs = gevo.benchmark_inputs(bench, n, seed)
    k0 = ob.Kernel(gevo.benchmark_ir(bench))
    ir = gevo.benchmark_ir(bench)
    threads = int(re.search(r"threads=(\d+)", ir).group(1))
    m = re.search(r"shared=(\d+)", ir)
    cfg = ob.config(threads, int(m.group(1)) if m else 0)
    tests = []
    for d in docs:
        doc = {"inputs": {k: {"type": b["type"], "data": b["data"]} for k, b in d["inputs"].items()},
               "scalars": d.get("scalars", {}), "oracle": {}}
        res = ob.execute(k0, ob.CTest(doc), cfg)
        doc["oracle"] = res["outputs"]
        tests.append(ob.CTest(doc))
    return tests, cfg


@pytest.mark.parametrize("bench,count,pick", [
    ("hot-branch", 160, None), ("bfs-load", 160, None), ("hot-memo", 96, None),
    ("lud-store", 96, None),
    # bench.py's own hot-branch sample: 748 is a 1000-trip loop per thread that
    # ends in a trap (partial jumps), 410 a budget spinner
    ("hot-branch", 1024, [748, 410, 874, 303] + list(range(0, 1024, 9))),
    ("nw-sync", 1024, [774, 415, 689, 852, 505] + list(range(1, 1024, 13)))])
def test_spinner_records_match_oracle(gevo, bench, count, pick):
    seed = gevo.train_seed(1)
    if pick is None:
        cands = gevo.sample_candidates(bench, count, 11, 4)
    else:
        every = gevo.sample_candidates(bench, count, 1, 4)
        cands = [every[i] for i in pick]
    suite = gevo.Suite.from_benchmark(bench, 2, seed)
    cfg = suite.exec_config()
    batch = suite.batch()
    for c in cands:
        batch.add_patch(c)
    gevo.spin_counters(reset=True)
    _, trec, _ = batch.eval(cfg, tests=True)
    jumped, _ = gevo.spin_counters()
    tests, ocfg = _oracle_tests(gevo, bench, 2, seed)
    orig = gevo.benchmark_ir(bench)
    budget_runs = 0
    for v, c in enumerate(cands):
        k = ob.Kernel(gevo.apply_patch(orig, c)[0])
        for t in range(2):
            exp = ob.execute(k, tests[t], ocfg)
            got = trec[v, t]
            where = (bench, v, t)
            assert STATUS[int(got["status"])] == exp["status"], where
            assert int(got["cost"]) == exp["cost"], where
            assert int(got["ir"]) == exp["ir"], where
            if exp["status"] != "completed":
                assert batch.reason(v, int(got["code"]), int(got["aux"])) == exp["reason"], where
            else:
                assert hex_double(float(got["error"])) == hex_double(exp["error"]), where
            budget_runs += exp["status"] == "budget"
    if bench in ("hot-branch", "bfs-load") and pick is None:
        assert budget_runs > 0 and jumped > 0
