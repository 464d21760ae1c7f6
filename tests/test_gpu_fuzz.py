"""Differential fuzzing beyond the golden fixtures: deeper random mutation
walks (up to 24 edits) of every corpus kernel, evaluated by the thread-parallel
and the sequential-lane interpreters and by the plain-C oracle (pinned to the
compiled reference in test_oracle.py), every (variant, test) record compared
field by field -- status, trap reason, cost, dynamic IR, error bits. The
budget is 20 000 instructions per thread for the large draws (the CPU oracle
stays fast while budget traps, spin-accelerator jumps and out-of-bounds traps
still occur) and the default 10^6 for a smaller draw."""
import pytest

import oracle_binding as ob
from _util import hex_double

pytestmark = pytest.mark.gpu

STATUS = {0: "completed", 1: "trap", 2: "budget"}
KERNELS = ["nw-sync", "lud-store", "hot-branch", "bfs-load", "lud-unroll", "hot-memo"]
BUDGET = 20_000


def _suite(gevo, name, n_tests, seed):
    ir = gevo.benchmark_ir(name)
    docs = gevo.benchmark_inputs(name, n_tests, seed)
    k0 = ob.Kernel(ir)
    threads = int(ir.split("threads=")[1].split()[0])
    shared = int(ir.split("shared=")[1].split()[0])
    tests = []
    for d in docs:
        doc = {"inputs": d["inputs"], "scalars": d.get("scalars", {}), "oracle": {}}
        res = ob.execute(k0, ob.CTest(doc), ob.config(threads, shared))
        assert res["status"] == "completed"
        doc["oracle"] = res["outputs"]
        tests.append(doc)
    return ir, tests, threads, shared


@pytest.mark.parametrize("budget,n", [(BUDGET, 400), (1_000_000, 100)])
@pytest.mark.parametrize("name", KERNELS)
def test_deep_walks_match_oracle(gevo, name, budget, n):
    ir, docs, threads, shared = _suite(gevo, name, 3, 777)
    suite = gevo.Suite.from_json(ir, docs)
    cfg = suite.exec_config().with_(budget=budget)
    cands = gevo.sample_candidates(name, n, 4242 + budget, 24)
    batch = suite.batch()
    for c in cands:
        batch.add_patch(c)
    _, tp, _ = batch.eval(cfg, tests=True)
    _, sq, _ = batch.eval(cfg, tests=True, sequential=True)
    for f in ("status", "code", "cost", "ir", "aux"):
        assert (tp[f] == sq[f]).all(), (name, f)
    ctests = [ob.CTest(d) for d in docs]
    ocfg = ob.config(threads, shared, budget)
    seen = set()
    for v, c in enumerate(cands):
        k = ob.Kernel(gevo.apply_patch(ir, c)[0])
        for t, ct in enumerate(ctests):
            exp = ob.execute(k, ct, ocfg)
            got = tp[v, t]
            where = (name, v, t)
            assert STATUS[int(got["status"])] == exp["status"], where
            assert int(got["cost"]) == exp["cost"] and int(got["ir"]) == exp["ir"], where
            if exp["status"] == "completed":
                assert hex_double(float(got["error"])) == hex_double(exp["error"]), where
            else:
                assert batch.reason(v, int(got["code"]), int(got["aux"])) == exp["reason"], where
            seen.add(exp["status"])
    assert "completed" in seen
