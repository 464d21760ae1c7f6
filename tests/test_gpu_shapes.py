"""Launch-shape edge cases: an empty batch, a single test, and simulated
thread counts beyond what one thread-parallel CTA holds (the host falls back
to the sequential-lane interpreter) -- records against the plain-C oracle."""
import pytest

import oracle_binding as ob
from _util import hex_double

pytestmark = pytest.mark.gpu
STATUS = {0: "completed", 1: "trap", 2: "budget"}


def _kernel(threads):
    # every thread writes s[tid] then, after a barrier, reads its neighbour's
    # word and stores the sum of both to out[tid]
    return """kernel wide(a: ptr<global> f32, out: ptr<global> f32, s: ptr<shared> f32) threads=%d shared=%d {
entry:
  %%0 = tid i32  #uid=0
  %%1 = load f32 a[%%0]  #uid=1
  store s[%%0], %%1  #uid=2
  sync  #uid=3
  %%2 = add i32 %%0, 1  #uid=4
  %%3 = nthreads i32  #uid=5
  %%4 = icmp.lt i32 %%2, %%3  #uid=6
  %%5 = select i32 %%4, %%2, 0  #uid=7
  %%6 = load f32 s[%%5]  #uid=8
  %%7 = fadd f32 %%1, %%6  #uid=9
  store out[%%0], %%7  #uid=10
  ret  #uid=11
}""" % (threads, threads)


def _doc(threads, seed):
    import random
    rnd = random.Random(seed)
    return {"inputs": {"a": {"type": "f32", "data": [rnd.random() for _ in range(threads)]},
                       "out": {"type": "f32", "data": [0.0] * threads}},
            "scalars": {}, "oracle": {}}


@pytest.mark.parametrize("threads", [33, 512, 700, 1024])
def test_thread_counts_match_oracle(gevo, threads):
    ir = _kernel(threads)
    docs = [_doc(threads, s) for s in range(3)]
    k = ob.Kernel(ir)
    for d in docs:
        d["oracle"] = ob.execute(k, ob.CTest(d), ob.config(threads, threads))["outputs"]
    # a mutant without the barrier (reads race: thread-id order decides) and
    # one reading past the shared region
    no_sync = ir.replace("  sync  #uid=3\n", "")
    oob = ir.replace("%5 = select i32 %4, %2, 0", "%5 = select i32 %4, %2, %3")
    suite = gevo.Suite.from_json(ir, docs)
    cfg = suite.exec_config()
    batch = suite.batch().add_ir(ir).add_ir(no_sync).add_ir(oob)
    _, tr, _ = batch.eval(cfg, tests=True)
    for v, text in enumerate((ir, no_sync, oob)):
        kv = ob.Kernel(text)
        for t, d in enumerate(docs):
            exp = ob.execute(kv, ob.CTest(d), ob.config(threads, threads))
            got = tr[v, t]
            where = (threads, v, t)
            assert STATUS[int(got["status"])] == exp["status"], where
            assert int(got["cost"]) == exp["cost"] and int(got["ir"]) == exp["ir"], where
            if exp["status"] == "completed":
                assert hex_double(float(got["error"])) == hex_double(exp["error"]), where
            else:
                assert batch.reason(v, int(got["code"]), int(got["aux"])) == exp["reason"], where


def test_empty_batch_and_single_test(gevo):
    suite = gevo.Suite.from_benchmark("hot-branch", 1, gevo.train_seed(1))
    cfg = suite.exec_config()
    vrec, tr, _ = suite.batch().eval(cfg, tests=True)
    assert len(vrec) == 0
    ir = gevo.benchmark_ir("hot-branch")
    batch = suite.batch().add_ir(ir)
    vrec, tr, _ = batch.eval(cfg, tests=True)
    assert tr.shape == (1, 1)
    assert int(tr[0, 0]["status"]) == 0 and bool(vrec[0]["accepted"])
    assert int(vrec[0]["execs_ref"]) == 1
