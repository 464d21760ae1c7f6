"""Thread-parallel interpreter (interp_tp_kernel: one lane per simulated
thread, same-phase conflict detection, re-run in thread-id order on a
conflict) against the sequential-lane interpreter and the plain-C oracle
(oracle/evoir_oracle.c, pinned to the reference's goldens). Every record
field is compared bit for bit."""
import json

import numpy as np
import pytest

import oracle_binding as ob
from _util import hex_double

pytestmark = pytest.mark.gpu

STATUS = {0: "completed", 1: "trap", 2: "budget"}
KERNELS = ("nw-sync", "bfs-load", "hot-branch", "hot-memo", "lud-store", "lud-unroll")


def _same(a, b):
    for f in ("status", "code", "cost", "ir", "aux"):
        if not np.array_equal(a[f], b[f]):
            bad = np.nonzero(a[f] != b[f])
            return "%s differs at %s" % (f, list(zip(*bad))[:5])
    done = a["status"] == 0
    if not np.array_equal(a["error"][done].view(np.uint64), b["error"][done].view(np.uint64)):
        return "error differs"
    return None


@pytest.mark.parametrize("bench", KERNELS)
def test_tp_matches_sequential_lanes_on_candidate_populations(gevo, bench):
    """Validated mutants (the search's raw candidate stream: traps, spinners,
    cross-thread races) x 16 tests, both interpreters, no early exit."""
    cands = gevo.sample_candidates(bench, 512, 5, 4)
    suite = gevo.Suite.from_benchmark(bench, 16, gevo.train_seed(1))
    cfg = suite.exec_config()
    batch = suite.batch()
    for c in cands:
        batch.add_patch(c)
    gevo.tp_counters(reset=True)
    _, tp, _ = batch.eval(cfg, tests=True)
    reruns, runs = gevo.tp_counters(reset=True)
    assert runs in (0, len(cands) * 16)  # 0: state too large for the on-chip kernel
    _, sq, _ = batch.eval(cfg, tests=True, sequential=True)
    assert _same(tp, sq) is None, (bench, _same(tp, sq))
    # the early-exit protocol yields the same verdicts
    v_tp, _, _ = batch.eval(cfg, early_exit=True)
    v_sq, _, _ = batch.eval(cfg, early_exit=True, sequential=True)
    for f in ("accepted", "failing_test", "code", "cost_mean", "error_max", "execs_ref", "ir_ref"):
        assert np.array_equal(v_tp[f], v_sq[f]), (bench, f)
    print(bench, "tp re-runs in id order:", reruns, "of", runs)


def test_tp_conflict_reruns_happen(gevo):
    """Across the corpus candidate streams some instances race across threads
    within a phase; those are re-run in thread-id order (and stay exact, see
    the test above)."""
    total = 0
    for bench in ("nw-sync", "lud-store", "bfs-load"):
        cands = gevo.sample_candidates(bench, 512, 5, 4)
        suite = gevo.Suite.from_benchmark(bench, 4, gevo.train_seed(1))
        batch = suite.batch()
        for c in cands:
            batch.add_patch(c)
        gevo.tp_counters(reset=True)
        batch.eval(suite.exec_config(), tests=True)
        total += gevo.tp_counters(reset=True)[0]
    assert total > 0


# Hand-written schedules: lowest stopping thread wins, higher threads abort.
STOP_KERNELS = {
    "trap3_spin_above": """kernel k(out: ptr<global> f32) threads=8 shared=0 {
entry:
  %0 = tid i32  #uid=0
  %1 = icmp.eq i32 %0, 3  #uid=1
  br %1, boom, next  #uid=2
next:
  %5 = icmp.lt i32 %0, 3  #uid=3
  br %5, done, loop  #uid=4
boom:
  %2 = sdiv i32 %0, 0  #uid=5
  ret  #uid=6
loop:
  %3 = phi f32 [0.0, next], [%4, loop]  #uid=7
  %4 = fadd f32 %3, 1.5  #uid=8
  br loop  #uid=9
done:
  store out[%0], 2.0  #uid=10
  ret  #uid=11
}""",
    "spin_below_trap": """kernel k(out: ptr<global> f32) threads=8 shared=0 {
entry:
  %0 = tid i32  #uid=0
  %1 = icmp.eq i32 %0, 3  #uid=1
  br %1, boom, loop  #uid=2
boom:
  %2 = sdiv i32 %0, 0  #uid=3
  ret  #uid=4
loop:
  %3 = phi f32 [0.0, entry], [%4, loop]  #uid=5
  %4 = fadd f32 %3, 1.5  #uid=6
  br loop  #uid=7
}""",
    "ring_read_same_phase": """kernel k(out: ptr<global> i32, s: ptr<shared> i32) threads=8 shared=8 {
entry:
  %0 = tid i32  #uid=0
  store s[%0], %0  #uid=1
  %1 = add i32 %0, 7  #uid=2
  %2 = sdiv i32 %1, 8  #uid=3
  %3 = mul i32 %2, 8  #uid=4
  %4 = sub i32 %1, %3  #uid=5
  %5 = load i32 s[%4]  #uid=6
  store out[%0], %5  #uid=7
  ret  #uid=8
}""",
    "ring_read_after_sync": """kernel k(out: ptr<global> i32, s: ptr<shared> i32) threads=8 shared=8 {
entry:
  %0 = tid i32  #uid=0
  store s[%0], %0  #uid=1
  sync  #uid=2
  %1 = add i32 %0, 7  #uid=3
  %2 = sdiv i32 %1, 8  #uid=4
  %3 = mul i32 %2, 8  #uid=5
  %4 = sub i32 %1, %3  #uid=6
  %5 = load i32 s[%4]  #uid=7
  store s[%0], %5  #uid=8
  store out[%0], %5  #uid=9
  ret  #uid=10
}""",
    # strided reads of a read-only buffer until they leave it: the spin
    # accelerator jumps to the iteration before the out-of-bounds load
    "stream_until_oob": """kernel k(a: ptr<global> f32, out: ptr<global> f32) threads=8 shared=0 {
entry:
  %0 = tid i32  #uid=0
  %1 = mul i32 %0, 1000  #uid=1
  br loop  #uid=2
loop:
  %2 = phi i32 [%1, entry], [%6, loop]  #uid=3
  %3 = phi f32 [0.0, entry], [%5, loop]  #uid=4
  %4 = load f32 a[%2]  #uid=5
  %5 = fadd f32 %3, %4  #uid=6
  %6 = add i32 %2, 3  #uid=7
  %7 = icmp.ne i32 %6, -5  #uid=8
  br %7, loop, done  #uid=9
done:
  store out[%0], %5  #uid=10
  ret  #uid=11
}""",
    # thread 0 spins reading and rewriting a word whose value changes every
    # iteration (path-irrelevant): the accelerator treats the load as varying
    "varying_word_spin": """kernel k(out: ptr<global> f32, s: ptr<shared> f32) threads=8 shared=8 {
entry:
  %0 = tid i32  #uid=0
  store s[%0], 1.0  #uid=1
  br loop  #uid=2
loop:
  %1 = phi i32 [0, entry], [%5, loop]  #uid=3
  %2 = load f32 s[%0]  #uid=4
  %3 = fadd f32 %2, 1.0  #uid=5
  store s[%0], %3  #uid=6
  %5 = add i32 %1, %0  #uid=7
  %6 = icmp.lt i32 %5, 50  #uid=8
  br %6, loop, done  #uid=9
done:
  store out[%0], %3  #uid=10
  ret  #uid=11
}""",
}


@pytest.mark.parametrize("name", sorted(STOP_KERNELS))
def test_tp_stop_and_race_schedules_match_oracle(gevo, name):
    ir = STOP_KERNELS[name]
    elem = "i32" if "i32" in ir.splitlines()[0] else "f32"
    zero = 0 if elem == "i32" else 0.0
    doc = {"inputs": {"out": {"type": elem, "data": [zero] * 8}}, "scalars": {}, "oracle": {}}
    budget = 20000
    if "a: ptr<global>" in ir:
        doc["inputs"]["a"] = {"type": "f32", "data": [0.5] * 30000}
        budget = 200000
    k = ob.Kernel(ir)
    ocfg = ob.config(8, 8 if "shared=8" in ir else 0, budget)
    exp = ob.execute(k, ob.CTest(doc), ocfg)
    if exp["status"] == "completed":
        doc["oracle"] = exp["outputs"]
        exp = ob.execute(k, ob.CTest(doc), ocfg)
    suite = gevo.Suite.from_json(ir, [json.dumps(doc)])
    cfg = suite.exec_config().with_(budget=budget)
    batch = suite.batch().add_ir(ir)
    for sequential in (False, True):
        _, trec, _ = batch.eval(cfg, tests=True, sequential=sequential)
        got = trec[0, 0]
        assert STATUS[int(got["status"])] == exp["status"], (name, sequential)
        assert int(got["cost"]) == exp["cost"], (name, sequential)
        assert int(got["ir"]) == exp["ir"], (name, sequential)
        if exp["status"] != "completed":
            assert batch.reason(0, int(got["code"]), int(got["aux"])) == exp["reason"]
        else:
            assert hex_double(float(got["error"])) == hex_double(exp["error"])
