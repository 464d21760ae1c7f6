"""Same-phase cross-thread memory patterns (no barrier between a write and a
read of another thread) on the thread-parallel interpreter against the
plain-C oracle, which runs the threads one after another like the reference:
RAW from lower threads with a conflict-free prefix (threads 0-3 private,
4-7 read 0-3's words), write-after-read only, reads that may observe a higher
thread's write (delay loops), and mixed patterns across several phases."""
import random

import pytest

import oracle_binding as ob
from _util import hex_double

pytestmark = pytest.mark.gpu
STATUS = {0: "completed", 1: "trap", 2: "budget"}

HEAD = """kernel k(a: ptr<global> i32, out: ptr<global> i32, s: ptr<shared> i32) threads=8 shared=16 {
entry:
  %0 = tid i32  #uid=0
  %1 = load i32 a[%0]  #uid=1
  %2 = add i32 %0, 8  #uid=2
  store s[%2], %1  #uid=3
  sync  #uid=4
"""

KERNELS = {
    # threads 0-3 work on their own word; 4-7 read the word of thread tid-4
    "prefix_raw": HEAD + """  %3 = mul i32 %1, 3  #uid=5
  store s[%0], %3  #uid=6
  %4 = sub i32 %0, 4  #uid=7
  %5 = icmp.lt i32 %0, 4  #uid=8
  %6 = select i32 %5, %0, %4  #uid=9
  %7 = load i32 s[%6]  #uid=10
  %8 = add i32 %7, %1  #uid=11
  store out[%0], %8  #uid=12
  ret  #uid=13
}""",
    # read the right neighbour's slot, then overwrite the own one (WAR only)
    "war_only": HEAD + """  %3 = add i32 %0, 9  #uid=5
  %4 = icmp.lt i32 %3, 16  #uid=6
  %5 = select i32 %4, %3, 8  #uid=7
  %6 = load i32 s[%5]  #uid=8
  %7 = add i32 %6, %1  #uid=9
  store s[%2], %7  #uid=10
  store out[%0], %7  #uid=11
  ret  #uid=12
}""",
    # write the own slot at once, spin a tid-dependent delay, then read the
    # right neighbour's slot (the reference shows its phase-start value)
    "late_read": HEAD + """  %3 = mul i32 %1, 5  #uid=5
  store s[%2], %3  #uid=6
  br spin  #uid=7
spin:
  %4 = phi i32 [0, entry], [%5, spin]  #uid=8
  %5 = add i32 %4, 1  #uid=9
  %6 = mul i32 %0, 3  #uid=10
  %7 = icmp.lt i32 %5, %6  #uid=11
  br %7, spin, done  #uid=12
done:
  %8 = add i32 %0, 9  #uid=13
  %9 = icmp.lt i32 %8, 16  #uid=14
  %10 = select i32 %9, %8, 8  #uid=15
  %11 = load i32 s[%10]  #uid=16
  %12 = add i32 %11, %5  #uid=17
  store out[%0], %12  #uid=18
  ret  #uid=19
}""",
    # a running sum through shared memory inside one phase (thread t reads
    # the slot thread t-1 writes; thread 0 reads thread 7's slot first), then
    # a barrier and a read-back
    "chain": HEAD + """  %3 = add i32 %0, 7  #uid=5
  %4 = icmp.lt i32 %0, 1  #uid=6
  %5 = select i32 %4, 15, %3  #uid=7
  %6 = load i32 s[%5]  #uid=8
  %7 = add i32 %6, %1  #uid=9
  store s[%2], %7  #uid=10
  sync  #uid=11
  %8 = load i32 s[%2]  #uid=12
  store out[%0], %8  #uid=13
  ret  #uid=14
}""",
}


def _doc(seed):
    rnd = random.Random(seed)
    return {"inputs": {"a": {"type": "i32", "data": [rnd.randrange(-1000, 1000) for _ in range(8)]},
                       "out": {"type": "i32", "data": [0] * 8}},
            "scalars": {}, "oracle": {}}


@pytest.mark.parametrize("name", sorted(KERNELS))
def test_same_phase_patterns_match_oracle(gevo, name):
    ir = KERNELS[name]
    k = ob.Kernel(ir)
    docs = [_doc(s) for s in range(4)]
    for d in docs:
        res = ob.execute(k, ob.CTest(d), ob.config(8, 16))
        assert res["status"] == "completed", (name, res["reason"])
        d["oracle"] = res["outputs"]
    suite = gevo.Suite.from_json(ir, docs)
    cfg = suite.exec_config()
    # the kernel itself plus mutants of it
    cands = gevo.sample_candidates_ir(ir, 60, 3, 4)
    batch = suite.batch().add_ir(ir)
    for c in cands:
        batch.add_patch(c)
    texts = [ir] + [gevo.apply_patch(ir, c)[0] for c in cands]
    for seq in (False, True):
        gevo.tp_counters(reset=True)
        _, tr, _ = batch.eval(cfg, tests=True, sequential=seq)
        if not seq and name in ("prefix_raw", "chain"):
            assert gevo.tp_counters(reset=True)[0] > 0  # the re-run path ran
        for v, text in enumerate(texts):
            kv = ob.Kernel(text)
            for t, d in enumerate(docs):
                exp = ob.execute(kv, ob.CTest(d), ob.config(8, 16))
                got = tr[v, t]
                where = (name, seq, v, t)
                assert STATUS[int(got["status"])] == exp["status"], where
                assert int(got["cost"]) == exp["cost"] and int(got["ir"]) == exp["ir"], where
                if exp["status"] == "completed":
                    assert hex_double(float(got["error"])) == hex_double(exp["error"]), where
                else:
                    assert batch.reason(v, int(got["code"]), int(got["aux"])) == exp["reason"], where
