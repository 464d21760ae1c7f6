"""GPU rank_population + select_best at the pool sizes of configs 4-5
(5 120 / 20 480 / 81 920) against the compiled reference's digests
(tests/golden/nsga_large.json, oracle/gen_golden_nsga_large.py): fronts,
front members in reference order, crowding distances (IEEE bytes) and the
select_best order, in four fitness distributions that drive every front
strategy of csrc/device/nsga_rank.cu (cost levels, error levels, staircase)."""
import importlib.util
import json
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "nsga_large.json")


def _gen():
    spec = importlib.util.spec_from_file_location(
        "gen_nsga_large", os.path.join(ROOT, "oracle", "gen_golden_nsga_large.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


CASES = json.load(open(GOLDEN))["cases"] if os.path.exists(GOLDEN) else []


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=lambda c: "%s-%d" % (c["dist"], c["n"]))
def test_rank_select_matches_reference_digests(gevo, case):
    g = _gen()
    cost, err = g.fits(case["dist"], case["n"])
    front, crowd, fronts = gevo.rank(cost, err)
    assert len(fronts) == case["n_fronts"]
    flat = np.array([i for f in fronts for i in f], np.int32)
    best, ms = gevo.select_best(cost, err, case["keep"])
    d = g.digests(front, crowd, flat, np.asarray(best, np.int32))
    assert d == case["digest"], (case["dist"], case["n"])


def test_oracle_rank_matches_reference_digests_small_pools():
    """The plain-C oracle's ranking pinned at the 5 120 pools too."""
    import oracle_binding as ob
    g = _gen()
    for case in CASES:
        if case["n"] != 5120:
            continue
        cost, err = g.fits(case["dist"], case["n"])
        front, crowd, fronts = ob.rank(cost, err)
        flat = np.array([i for f in fronts for i in f], np.int32)
        d = g.digests(np.asarray(front, np.int32), np.asarray(crowd, np.float64), flat,
                      np.zeros(0, np.int32))
        assert d["front"] == case["digest"]["front"], case["dist"]
        assert d["crowding"] == case["digest"]["crowding"], case["dist"]
        assert d["fronts"] == case["digest"]["fronts"], case["dist"]
