"""Suites larger than one thread-parallel test group (40 and 70 tests: the
CTA covers at most 32 tests, so a variant's tests span two or three CTAs and
the early-exit protocol crosses them). Per-test records of the thread-parallel
interpreter against the sequential-lane interpreter, and each variant's
evaluate_fitness verdict (accepted, failing test, reference-equivalent
executions and dynamic IR, cost mean, error max) against the plain-C oracle."""
import pytest

import oracle_binding as ob
from _util import hex_double

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_tests", [40, 70])
@pytest.mark.parametrize("name", ["nw-sync", "hot-branch", "bfs-load"])
def test_multi_group_suites(gevo, name, n_tests):
    ir = gevo.benchmark_ir(name)
    docs = gevo.benchmark_inputs(name, n_tests, 31337)
    threads = int(ir.split("threads=")[1].split()[0])
    shared = int(ir.split("shared=")[1].split()[0])
    k0 = ob.Kernel(ir)
    tests = []
    for d in docs:
        doc = {"inputs": d["inputs"], "scalars": d.get("scalars", {}), "oracle": {}}
        res = ob.execute(k0, ob.CTest(doc), ob.config(threads, shared))
        doc["oracle"] = res["outputs"]
        tests.append(doc)
    # a wrong oracle word in a test of the second group: every variant that
    # passes the first group fails there, and the tests after it are skipped
    bad = tests[35]["oracle"]
    first = sorted(bad)[0]
    h = bad[first]["hex"]
    bad[first] = {"type": bad[first]["type"], "hex": "3f800000" + h[8:] if h[:8] != "3f800000"
                  else "40000000" + h[8:]}
    suite = gevo.Suite.from_json(ir, tests)
    budget = 50_000
    cfg = suite.exec_config().with_(budget=budget)
    cands = gevo.sample_candidates(name, 48, 99, 6)
    batch = suite.batch()
    batch.add_ir(ir)
    for c in cands:
        batch.add_patch(c)
    _, tp, _ = batch.eval(cfg, tests=True)
    _, sq, _ = batch.eval(cfg, tests=True, sequential=True)
    for f in ("status", "code", "cost", "ir", "aux", "error"):
        assert (tp[f] == sq[f]).all(), (name, f)
    ctests = [ob.CTest(d) for d in tests]
    ocfg = ob.config(threads, shared, budget)
    late = 0
    for tol in (0.0, 0.01):
        vrec, _, _ = batch.eval(cfg, tolerance=tol, early_exit=True)
        late += int((vrec["failing_test"] >= 32).sum())
        for v, text in enumerate([ir] + [gevo.apply_patch(ir, c)[0] for c in cands]):
            exp = ob.evaluate_fitness(ob.Kernel(text), ctests, ocfg, tol)
            got = vrec[v]
            where = (name, n_tests, tol, v)
            assert bool(got["accepted"]) == exp["accepted"], where
            assert int(got["failing_test"]) == exp["failing_test"], where
            assert int(got["execs_ref"]) == exp["execs_ref"], where
            assert int(got["ir_ref"]) == exp["ir_ref"], where
            if exp["accepted"]:
                assert hex_double(float(got["cost_mean"])) == hex_double(exp["cost"]), where
                assert hex_double(float(got["error_max"])) == hex_double(exp["error"]), where
    assert late >= 2  # the cross-group early exit was exercised
