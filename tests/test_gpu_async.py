"""Concurrent resident-batch evaluation (gevo_eval_resident_async / _wait):
several batches in flight on their own streams give exactly the records of
the synchronous path, with and without the in-call bytecode upload."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
FIELDS = ("accepted", "failing_test", "code", "cost_mean", "error_max", "execs_ref", "ir_ref", "aux")


def test_async_batches_match_sync(gevo):
    ks = ("hot-branch", "nw-sync", "bfs-load", "hot-memo")
    batches, cfgs, want = {}, {}, {}
    for k in ks:
        suite = gevo.Suite.from_benchmark(k, 16, gevo.train_seed(1))
        cfgs[k] = suite.exec_config()
        b = suite.batch()
        for c in gevo.sample_candidates(k, 384, 9, 4):
            b.add_patch(c)
        b.make_resident()
        batches[k] = (suite, b)
        want[k], _ = b.eval_resident(cfgs[k], tolerance=0.01, early_exit=True, records=True)
    for upload in (False, True, False):
        for k in ks:
            batches[k][1].eval_resident_async(cfgs[k], tolerance=0.01, early_exit=True,
                                              upload=upload)
        for k in ks:
            got, st = batches[k][1].wait(records=True)
            assert st.launches > 0
            assert (st.h2d_bytes > 0) == upload
            for f in FIELDS:
                assert np.array_equal(got[f], want[k][f]), (k, f, upload)


def test_resident_batch_grows_after_upload(gevo):
    """A resident batch page-locks its host bytecode for in-call uploads;
    adding variants afterwards (the blob reallocates) must drop that
    registration first and give the records of a fresh batch."""
    suite = gevo.Suite.from_benchmark("nw-sync", 8, gevo.train_seed(1))
    cfg = suite.exec_config()
    cands = gevo.sample_candidates("nw-sync", 600, 21, 4)
    b = suite.batch()
    for c in cands[:100]:
        b.add_patch(c)
    for round_ in range(3):
        b.eval_resident_async(cfg, tolerance=0.0, early_exit=True, upload=True)
        got, _ = b.wait(records=True)
        fresh = suite.batch()
        for c in cands[:len(got)]:
            fresh.add_patch(c)
        want, _, _ = fresh.eval(cfg, tolerance=0.0, early_exit=True)
        for f in FIELDS:
            assert np.array_equal(got[f], want[f]), (round_, f)
        for c in cands[100 + 200 * round_:300 + 200 * round_]:
            b.add_patch(c)
    del b  # registration released before the blob
