"""Non-default cycle-cost tables (ExecConfig::cost_table, src/vm.cpp:12-30):
per-launch block costs and suffix refunds (block_cost_kernel) must follow the
table, including zero and large entries, on trapping, budget-bound and
completing mutants -- records against the plain-C oracle."""
import random

import pytest

import oracle_binding as ob
from _util import hex_double

pytestmark = pytest.mark.gpu
STATUS = {0: "completed", 1: "trap", 2: "budget"}


@pytest.mark.parametrize("name", ["nw-sync", "bfs-load", "hot-memo"])
def test_random_cost_tables_match_oracle(gevo, name):
    rnd = random.Random(hash(name) & 0xFFFF)
    ir = gevo.benchmark_ir(name)
    threads = int(ir.split("threads=")[1].split()[0])
    shared = int(ir.split("shared=")[1].split()[0])
    docs = gevo.benchmark_inputs(name, 2, 5150)
    k0 = ob.Kernel(ir)
    tests = []
    for d in docs:
        doc = {"inputs": d["inputs"], "scalars": d.get("scalars", {}), "oracle": {}}
        doc["oracle"] = ob.execute(k0, ob.CTest(doc), ob.config(threads, shared))["outputs"]
        tests.append(doc)
    suite = gevo.Suite.from_json(ir, tests)
    cands = gevo.sample_candidates(name, 64, 7, 8)
    batch = suite.batch().add_ir(ir)
    for c in cands:
        batch.add_patch(c)
    texts = [ir] + [gevo.apply_patch(ir, c)[0] for c in cands]
    ctests = [ob.CTest(d) for d in tests]
    for trial in range(3):
        costs = [rnd.choice([0, 1, 2, 3, 7, 20, 1000]) for _ in range(14)]
        budget = rnd.choice([5_000, 100_000])
        cfg = suite.exec_config().with_(budget=budget, costs=costs)
        _, tr, _ = batch.eval(cfg, tests=True)
        ocfg = ob.config(threads, shared, budget, costs)
        for v, text in enumerate(texts):
            kv = ob.Kernel(text)
            for t, ct in enumerate(ctests):
                exp = ob.execute(kv, ct, ocfg)
                got = tr[v, t]
                where = (name, trial, v, t, costs)
                assert STATUS[int(got["status"])] == exp["status"], where
                assert int(got["cost"]) == exp["cost"] and int(got["ir"]) == exp["ir"], where
                if exp["status"] == "completed":
                    assert hex_double(float(got["error"])) == hex_double(exp["error"]), where
