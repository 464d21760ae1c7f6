"""Parity of the sm_100a path against the compiled reference (tests/golden/,
produced by oracle/ref_dump.cpp from /root/reference/proj). Every check is
bit-exact: status, reason string, cycle cost, dynamic IR count, output bits
(NaN payloads canonicalised), error and fitness doubles,
Pareto fronts, crowding distances, selection order, and whole search
trajectories (log.csv / report.json bytes)."""
import json
import os

import pytest

from _util import STATUS_NAME, fixture_test_json, hex_double, outputs_hash

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _status(rec):
    return STATUS_NAME[int(rec["status"])]


def test_trap_classes_and_semantics(gevo, vmcases_golden):
    """Every interpreter trap class and the value/memory semantics cases."""
    for case in vmcases_golden:
        ir = case["ir"]
        test = fixture_test_json(case["test"])
        suite = gevo.Suite.from_json(ir, [test])
        cfg = suite.exec_config().with_(budget=case["budget"])
        batch = suite.batch().add_ir(ir)
        _, trec, _ = batch.eval(cfg, tests=True)
        r = trec[0, 0]
        exp = case["exec"]
        assert _status(r) == exp["status"], case["label"]
        reason = "" if r["status"] == 0 else batch.reason(0, int(r["code"]), int(r["aux"]))
        assert reason == exp["reason"], case["label"]
        assert int(r["cost"]) == exp["cost"], case["label"]
        assert int(r["ir"]) == exp["ir"], case["label"]
        if exp["status"] == "completed":
            assert hex_double(float(r["error"])) == exp["err"], case["label"]
            outs = batch.outputs(cfg)[0][0]
            assert outputs_hash(outs) == exp["out"], case["label"]
        # batch-of-one evoir::execute / evaluate_fitness entry points
        res = gevo.execute(ir, test, cfg)
        assert res["status"] == exp["status"] and res["reason"] == exp["reason"]
        assert res["cost"] == exp["cost"], case["label"]
        out = gevo.evaluate_fitness(ir, [test], cfg, 0.0)
        want = case["outcome"]
        assert out["accepted"] == want["accepted"], case["label"]
        assert out["failing_test"] == want["failing_test"], case["label"]
        assert out["reason"] == want["reason"], case["label"]
        assert out["cost"] == want["cost"] and out["error"] == want["error"], case["label"]


def test_corpus_kernels_on_generated_suites(gevo, corpus_golden):
    """Original and hand-improved kernels on the config-1/2 suites."""
    tests = {}
    for j in corpus_golden:
        if j["kind"] == "test":
            tests.setdefault((j["name"], j["suite"]), []).append(j)
    kernels = {j["name"]: j for j in corpus_golden if j["kind"] == "kernel"}
    for (name, label), recs in sorted(tests.items()):
        recs.sort(key=lambda r: r["index"])
        ir = kernels[name]["ir"]
        suite = gevo.Suite.from_json(ir, [fixture_test_json(r["test"]) for r in recs])
        cfg = suite.exec_config()
        batch = suite.batch().add_ir(ir).add_ir(kernels[name]["improved"])
        _, trec, _ = batch.eval(cfg, tests=True)
        outs = batch.outputs(cfg)
        for v, key in enumerate(("orig", "improved")):
            for t, r in enumerate(recs):
                exp = r[key]
                got = trec[v, t]
                assert _status(got) == exp["status"], (name, label, key, t)
                assert int(got["cost"]) == exp["cost"], (name, label, key, t)
                assert int(got["ir"]) == exp["ir"], (name, label, key, t)
                assert hex_double(float(got["error"])) == exp["err"], (name, label, key, t)
                assert outputs_hash(outs[v][t]) == exp["out"], (name, label, key, t)


def test_generated_suites_match_reference(gevo, corpus_golden):
    """generate_tests (inputs on the host, oracles from a device batch) is
    bit-identical: the suite built by the product evaluates the reference
    oracle files with error exactly 0 for the original kernel."""
    for j in corpus_golden:
        if j["kind"] != "test" or j["suite"] != "train3_seed1":
            continue
        mine = gevo.benchmark_inputs(j["name"], 3, j["seed"])[j["index"]]
        ref = fixture_test_json(j["test"])
        for n, b in ref["inputs"].items():
            words = b["hex"]
            got = mine["inputs"][n]
            assert got["type"] == b["type"]
            import struct
            fmt = "<i" if b["type"] == "i32" else "<f"
            packed = "".join("%08x" % struct.unpack("<I", struct.pack(fmt, x))[0]
                             for x in got["data"])
            assert packed == words, (j["name"], n)


def _mutant_parity(gevo, records, budget):
    by_kernel = {}
    for m in records:
        if "tests" in m:
            by_kernel.setdefault(m["name"], []).append(m)
    checked = 0
    for name, ms in sorted(by_kernel.items()):
        suite = gevo.Suite.from_benchmark(name, 3, 4242)
        cfg = suite.exec_config().with_(budget=budget)
        batch = suite.batch()
        for m in ms:
            batch.add_patch(m["parent_patch"] + [m["edit"]])
        _, trec, _ = batch.eval(cfg, tests=True)
        outs = batch.outputs(cfg)
        for v, m in enumerate(ms):
            for t, exp in enumerate(m["tests"]):
                got = trec[v, t]
                where = (name, m["i"], t)
                assert _status(got) == exp["status"], where
                reason = "" if got["status"] == 0 else batch.reason(v, int(got["code"]),
                                                                    int(got["aux"]))
                assert reason == exp["reason"], where
                assert int(got["cost"]) == exp["cost"], where
                assert int(got["ir"]) == exp["ir"], where
                if exp["status"] == "completed":
                    assert hex_double(float(got["error"])) == exp["err"], where
                    assert outputs_hash(outs[v][t]) == exp["out"], where
                checked += 1
        for tol, key in ((0.0, "outcome0"), (0.01, "outcome01")):
            vrec, _, _ = batch.eval(cfg, tolerance=tol, early_exit=True)
            for v, m in enumerate(ms):
                exp, got = m[key], vrec[v]
                where = (name, m["i"], key)
                assert bool(got["accepted"]) == exp["accepted"], where
                assert int(got["failing_test"]) == exp["failing_test"], where
                if exp["accepted"]:
                    assert hex_double(float(got["cost_mean"])) == exp["cost"], where
                    assert hex_double(float(got["error_max"])) == exp["error"], where
                else:
                    reason = batch.reason(v, int(got["code"]), int(got["aux"]),
                                          float(got["fail_error"]))
                    assert reason == exp["reason"], where
    return checked


def test_mutant_population_full_budget(gevo, mutants_golden):
    """Seeded random-walk mutants (valid and invalid, trapping, spinning) at
    the default 10^6 instruction budget."""
    assert _mutant_parity(gevo, mutants_golden, 1_000_000) > 3000


def test_mutant_population_reduced_budget(gevo, mutants_budget_golden):
    assert _mutant_parity(gevo, mutants_budget_golden, 20_000) > 1000


def test_nsga_rank_and_selection(gevo, nsga_golden):
    import struct
    for case in nsga_golden:
        cost = [struct.unpack("<d", bytes.fromhex(c)[::-1])[0] for c, _ in case["fits"]]
        err = [struct.unpack("<d", bytes.fromhex(e)[::-1])[0] for _, e in case["fits"]]
        front, crowd, fronts = gevo.rank(cost, err)
        assert fronts == case["fronts"]
        assert [hex_double(float(x)) for x in crowd] == case["crowding"]
        best, tour = gevo.nsga_select(cost, err, case["keep"], int(case["tseed"], 16),
                                      len(cost))
        assert best == case["select_best"]
        assert tour == case["tournament"]


RUNS = sorted(os.listdir(os.path.join(GOLDEN, "runs"))) if os.path.isdir(
    os.path.join(GOLDEN, "runs")) else []


def _run_args(name):
    # config1_<bench> | small_<bench>_<mode> | config2_<bench>
    if name.startswith("config1_"):
        return name[len("config1_"):], 1, 32, 5, "default", 3, 3
    if name.startswith("config2_"):
        bench = name[len("config2_"):]
        mode = "mo" if bench == "hot-memo" else "default"
        return bench, 1, 256, 50, mode, 16, 3
    bench, mode = name[len("small_"):].rsplit("_", 1)
    return bench, (7 if mode == "default" else 3), 16, 4, mode, 3, 2


@pytest.mark.parametrize("run", [r for r in RUNS if not r.startswith("config2_")])
def test_search_trajectory_bytes(gevo, run):
    bench, seed, pop, gens, mode, train, held = _run_args(run)
    log, rep, st = gevo.run_search(bench, seed, pop, gens, mode, -1.0, train, held, jobs=4)
    d = os.path.join(GOLDEN, "runs", run)
    assert log == open(os.path.join(d, "log.csv")).read()
    # the report echoes the host thread count; the reference run used jobs=1
    assert rep.replace('"jobs": 4,', '"jobs": 1,') == open(os.path.join(d, "report.json")).read()
    assert st.executions > 0 and st.launches > 0


@pytest.mark.slow
@pytest.mark.parametrize("run", [r for r in RUNS if r.startswith("config2_")])
def test_config2_trajectory_bytes(gevo, run):
    bench, seed, pop, gens, mode, train, held = _run_args(run)
    log, rep, st = gevo.run_search(bench, seed, pop, gens, mode, -1.0, train, held, jobs=8)
    d = os.path.join(GOLDEN, "runs", run)
    assert log == open(os.path.join(d, "log.csv")).read()
    ref = open(os.path.join(d, "report.json")).read()
    jobs = json.loads(ref)["config"]["jobs"]
    assert rep.replace('"jobs": 8,', '"jobs": %d,' % jobs) == ref
