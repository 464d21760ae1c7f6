"""Pins the plain-C oracle (oracle/evoir_oracle.c) to the compiled reference's
golden vectors before any parity test trusts it. CPU only."""
import json
import os
import struct

import pytest

import oracle_binding as ob
from _util import fixture_test_json, hex_double, outputs_hash


def _cfg_for(kernel_ir, budget=1_000_000, costs=None):
    head = kernel_ir.split("\n", 1)[0]
    threads = int(head.split("threads=")[1].split()[0])
    shared = int(head.split("shared=")[1].split()[0])
    if costs is None:
        return ob.config(threads, shared, budget)
    return ob.config(threads, shared, budget, costs)


def test_oracle_vmcases(vmcases_golden):
    for case in vmcases_golden:
        k = ob.Kernel(case["ir"])
        t = ob.CTest(fixture_test_json(case["test"]))
        r = ob.execute(k, t, _cfg_for(case["ir"], case["budget"]))
        exp = case["exec"]
        assert (r["status"], r["reason"], r["cost"], r["ir"]) == (
            exp["status"], exp["reason"], exp["cost"], exp["ir"]), case["label"]
        if exp["status"] == "completed":
            assert hex_double(r["error"]) == exp["err"], case["label"]
            assert outputs_hash(r["outputs"]) == exp["out"], case["label"]
        o = ob.evaluate_fitness(k, [t], _cfg_for(case["ir"], case["budget"]), 0.0)
        want = case["outcome"]
        assert o["accepted"] == want["accepted"] and o["reason"] == want["reason"], case["label"]
        assert o["failing_test"] == want["failing_test"]
        assert hex_double(o["cost"]) == want["cost"] and hex_double(o["error"]) == want["error"]


def test_oracle_corpus_suites(corpus_golden):
    kernels = {j["name"]: j for j in corpus_golden if j["kind"] == "kernel"}
    n = 0
    for j in corpus_golden:
        if j["kind"] != "test" or j["suite"] != "train3_seed1":
            continue
        t = ob.CTest(fixture_test_json(j["test"]))
        for key, ir in (("orig", kernels[j["name"]]["ir"]), ("improved",
                                                             kernels[j["name"]]["improved"])):
            r = ob.execute(ob.Kernel(ir), t, _cfg_for(ir))
            exp = j[key]
            assert (r["status"], r["cost"], r["ir"]) == (exp["status"], exp["cost"], exp["ir"])
            assert hex_double(r["error"]) == exp["err"]
            assert outputs_hash(r["outputs"]) == exp["out"]
            n += 1
    assert n == 36


def test_oracle_mutants_reduced_budget(gevo, mutants_budget_golden):
    """Mutant executions (the product's host apply_patch is itself pinned by
    kernel_hash in test_host_parity) against reference records."""
    names = gevo.benchmark_names()
    orig = {n: gevo.benchmark_ir(n) for n in names}
    tests = {}
    checked = 0
    for m in mutants_budget_golden:
        if "tests" not in m:
            continue
        name = m["name"]
        if name not in tests:
            docs = gevo.benchmark_inputs(name, 3, 4242)
            tests[name] = docs
        ir, _ = gevo.apply_patch(orig[name], m["parent_patch"] + [m["edit"]])
        k = ob.Kernel(ir)
        for ti, exp in enumerate(m["tests"]):
            if exp["status"] == "budget" and ti > 0:
                continue  # keep the CPU suite short; budget cases covered at ti == 0
            # oracle buffers are the original's outputs on the same inputs
            doc = dict(tests[name][ti])
            base = ob.execute(ob.Kernel(orig[name]), ob.CTest(doc), _cfg_for(ir, 20000))
            outs = {s: base["outputs"][s] for s in base["outputs"]}
            doc = {"inputs": doc["inputs"], "scalars": doc.get("scalars", {}),
                   "oracle": {s: outs[s] for s in outs if _is_output(name, s)}}
            r = ob.execute(k, ob.CTest(doc), _cfg_for(ir, 20000))
            assert (r["status"], r["reason"], r["cost"], r["ir"]) == (
                exp["status"], exp["reason"], exp["cost"], exp["ir"]), (name, m["i"], ti)
            if exp["status"] == "completed":
                assert hex_double(r["error"]) == exp["err"], (name, m["i"], ti)
                assert outputs_hash(r["outputs"]) == exp["out"], (name, m["i"], ti)
            checked += 1
    assert checked > 500


def _is_output(bench, name):
    corpus = os.path.join(ob.ROOT, "paper_2004_08140_b200", "data", "corpus.json")
    for b in json.load(open(corpus))["benchmarks"]:
        if b["name"] == bench:
            return any(x["name"] == name and x.get("output") for x in b["buffers"])
    return False


def test_oracle_nsga(nsga_golden):
    for case in nsga_golden:
        cost = [struct.unpack(">d", bytes.fromhex(c))[0] for c, _ in case["fits"]]
        err = [struct.unpack(">d", bytes.fromhex(e))[0] for _, e in case["fits"]]
        _, crowd, fronts = ob.rank(cost, err)
        assert fronts == case["fronts"]
        assert [hex_double(float(x)) for x in crowd] == case["crowding"]
        assert ob.select_best(cost, err, case["keep"]) == case["select_best"]


@pytest.mark.parametrize("name", ["svm-rbf", "conv-bn"])
def test_oracle_authored_kernels(gevo, name):
    """Authored config-3/4 kernels (reduced sizes): the oracle reproduces the
    compiled reference's per-test records for the original and 40 mutants."""
    from conftest import authored_fixture
    head, recs = authored_fixture(name)
    ir, _ = gevo.authored_kernel(name)
    gen = json.dumps(head["gen"])
    docs = gevo.spec_inputs(gen, head["n_tests"], head["seed"])
    k0 = ob.Kernel(ir)
    cfg = _cfg_for(ir, head["budget"])
    tests = []
    for d in docs:
        doc = {"inputs": d["inputs"], "scalars": d.get("scalars", {}), "oracle": {}}
        res = ob.execute(k0, ob.CTest(doc), cfg)
        doc["oracle"] = res["outputs"]
        tests.append(ob.CTest(doc))
    for rec in recs:
        k = ob.Kernel(gevo.apply_patch(ir, json.dumps(rec["patch"]))[0])
        for t, exp in zip(tests, rec["tests"]):
            r = ob.execute(k, t, cfg)
            where = (name, rec["i"])
            assert (r["status"], r["reason"], r["cost"], r["ir"]) == (
                exp["status"], exp["reason"], exp["cost"], exp["ir"]), where
            if exp["status"] == "completed":
                assert hex_double(r["error"]) == exp["err"], where
                assert outputs_hash(r["outputs"]) == exp["out"], where
