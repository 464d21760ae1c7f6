"""N>1 host path on CPU: world-size-2 gloo process group, the same sharding and
fitness all-gather bench.py runs over NCCL, checked against the oracle's
rank_population (oracle/liboracle.so, test infrastructure only)."""
import os
import socket

import numpy as np
import pytest

from paper_2004_08140_b200 import dist as gdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_range_partitions():
    for n in (0, 1, 7, 1024, 1025):
        for world in (1, 2, 3, 8):
            spans = [gdist.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _population(n, seed):
    rng = np.random.default_rng(seed)
    rows = np.empty((n, 3))
    rows[:, 0] = rng.integers(100, 140, n) * 8.0
    rows[:, 1] = np.where(rng.random(n) < 0.5, 0.0, rng.random(n) * 0.02)
    rows[:, 2] = (rng.random(n) < 0.7).astype(float)
    return rows


def _worker(rank, world, port, n, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = _population(n, 7)
        b, e = gdist.shard_range(n, rank, world)
        got = gdist.allgather_fitness(full[b:e])
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [1023, 64])
def test_allgather_fitness_world2_matches_oracle_rank(n):
    import multiprocessing as mp
    import oracle_binding as ob

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = _population(n, 7)
    for r in range(2):
        assert res[r].shape == full.shape
        assert np.array_equal(res[r], full)  # bit-exact, batch order
    cost, err, idx = gdist.accepted_fitness(res[0])
    keep = full[:, 2] > 0.5
    assert np.array_equal(idx, np.nonzero(keep)[0])
    # the gathered population ranks exactly like the unsharded one
    f_all, c_all, fronts_all = ob.rank(full[keep, 0], full[keep, 1])
    f_g, c_g, fronts_g = ob.rank(cost, err)
    assert fronts_all == fronts_g
    assert np.array_equal(np.asarray(c_all).view(np.uint64), np.asarray(c_g).view(np.uint64))
