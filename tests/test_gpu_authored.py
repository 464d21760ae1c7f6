"""Authored workload kernels of BASELINE.json configs 3 and 4 (SVM RBF kernel
row on a9a-shaped data, conv3x3 + batch-norm on CIFAR-shaped tensors,
paper_2004_08140_b200/data/kernels/) on the device: thread-parallel
interpreter (256 simulated threads, instance memory in global cells) against
the sequential-lane interpreter and the plain-C oracle, every record field bit
for bit. Reduced sizes keep the CPU oracle fast; one larger case per kernel
runs the original kernel at (near) full size."""
import json

import numpy as np
import pytest

import oracle_binding as ob
from _util import hex_double

pytestmark = pytest.mark.gpu
STATUS = {0: "completed", 1: "trap", 2: "budget"}


def _resize(name, gen_json, scale):
    g = json.loads(gen_json)
    if name == "svm-rbf":
        rows = scale
        for b in g["buffers"]:
            if b["name"] == "X":
                b["size"] = rows * 123
            if b["name"] == "K":
                b["size"] = rows
        for sc in g["scalars"]:
            if sc["name"] == "n":
                sc["value"] = rows
    else:
        total = scale
        for b in g["buffers"]:
            if b["name"] == "out":
                b["size"] = total
        for sc in g["scalars"]:
            if sc["name"] == "total":
                sc["value"] = total
    return json.dumps(g)


def _oracle_suite(gevo, ir, gen, n, seed):
    docs = gevo.spec_inputs(gen, n, seed)
    k0 = ob.Kernel(ir)
    cfg = ob.config(256, 0)
    tests = []
    for d in docs:
        doc = {"inputs": d["inputs"], "scalars": d.get("scalars", {}), "oracle": {}}
        res = ob.execute(k0, ob.CTest(doc), cfg)
        assert res["status"] == "completed"
        doc["oracle"] = res["outputs"]
        tests.append(ob.CTest(doc))
    return tests, cfg


@pytest.mark.parametrize("name,scale", [("svm-rbf", 40), ("conv-bn", 1024)])
def test_authored_mutants_match_oracle(gevo, name, scale):
    ir, gen = gevo.authored_kernel(name)
    gen = _resize(name, gen, scale)
    seed = 7
    suite = gevo.Suite.from_spec(ir, gen, 2, seed)
    cfg = suite.exec_config().with_(budget=200_000)
    cands = gevo.sample_candidates_ir(ir, 24, 3, 3)
    batch = suite.batch()
    for c in cands:
        batch.add_patch(c)
    _, tp, _ = batch.eval(cfg, tests=True)
    _, sq, _ = batch.eval(cfg, tests=True, sequential=True)
    for f in ("status", "code", "cost", "ir", "aux"):
        assert np.array_equal(tp[f], sq[f]), (name, f)
    tests, ocfg = _oracle_suite(gevo, ir, gen, 2, seed)
    ocfg = ob.config(256, 0, 200_000)
    for v, c in enumerate(cands):
        k = ob.Kernel(gevo.apply_patch(ir, c)[0])
        for t in range(2):
            exp = ob.execute(k, tests[t], ocfg)
            got = tp[v, t]
            where = (name, v, t)
            assert STATUS[int(got["status"])] == exp["status"], where
            assert int(got["cost"]) == exp["cost"] and int(got["ir"]) == exp["ir"], where
            if exp["status"] == "completed":
                assert hex_double(float(got["error"])) == hex_double(exp["error"]), where
            else:
                assert batch.reason(v, int(got["code"]), int(got["aux"])) == exp["reason"], where


@pytest.mark.parametrize("name,scale", [("svm-rbf", 2048), ("conv-bn", 8192)])
def test_authored_original_large(gevo, name, scale):
    ir, gen = gevo.authored_kernel(name)
    gen = _resize(name, gen, scale)
    suite = gevo.Suite.from_spec(ir, gen, 1, 11)
    batch = suite.batch().add_ir(ir)
    _, tp, _ = batch.eval(suite.exec_config(), tests=True)
    tests, ocfg = _oracle_suite(gevo, ir, gen, 1, 11)
    exp = ob.execute(ob.Kernel(ir), tests[0], ocfg)
    got = tp[0, 0]
    assert exp["status"] == "completed" and int(got["status"]) == 0
    assert int(got["cost"]) == exp["cost"] and int(got["ir"]) == exp["ir"]
    assert float(got["error"]) == 0.0 == exp["error"]


@pytest.mark.parametrize("name", ["svm-rbf", "conv-bn", "full_svm-rbf", "full_conv-bn"])
def test_authored_golden_records(gevo, name):
    """Device records and verdicts against the compiled reference's fixture
    (oracle/gen_golden_authored.py). The full_* fixtures are the BASELINE
    shapes (a9a X[32561x123] -> K[32561]; CIFAR in[3x32x32] -> out[64x32x32])
    with 256 mutants + the original, budget 1e6, tolerance 0.01."""
    from conftest import authored_fixture
    head, recs = authored_fixture(name)
    name = name.replace("full_", "")
    ir, _ = gevo.authored_kernel(name)
    suite = gevo.Suite.from_spec(ir, json.dumps(head["gen"]), head["n_tests"], head["seed"])
    cfg = suite.exec_config().with_(budget=head["budget"])
    batch = suite.batch()
    for rec in recs:
        batch.add_patch(json.dumps(rec["patch"]))
    vr, tr, _ = batch.eval(cfg, tolerance=head["tol"], tests=True)
    for v, rec in enumerate(recs):
        for t, exp in enumerate(rec["tests"]):
            got = tr[v, t]
            where = (name, rec["i"], t)
            assert STATUS[int(got["status"])] == exp["status"], where
            assert int(got["cost"]) == exp["cost"] and int(got["ir"]) == exp["ir"], where
            if exp["status"] == "completed":
                assert hex_double(float(got["error"])) == exp["err"], where
            else:
                assert batch.reason(v, int(got["code"]), int(got["aux"])) == exp["reason"], where
        assert bool(vr[v]["accepted"]) == rec["outcome"]["accepted"], (name, rec["i"])
        assert int(vr[v]["failing_test"]) == rec["outcome"]["failing_test"], (name, rec["i"])
        if rec["outcome"]["accepted"]:
            assert hex_double(float(vr[v]["cost_mean"])) == rec["outcome"]["cost"]
            assert hex_double(float(vr[v]["error_max"])) == rec["outcome"]["error"]
