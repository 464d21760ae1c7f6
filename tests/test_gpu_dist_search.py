"""Multi-rank search: two or four processes share one GPU here
(the driver's boxes have one), each evaluates its shard of every candidate
batch (contiguous shards cut at equal predicted cost), and the per-variant
records are all-gathered over a gloo group through the collective callback.
The in-library NCCL exchange (gevo_set_nccl: ncclAllGather on the device
record buffers, one process per GPU) runs here at world 1 -- NCCL refuses two
ranks on one device. Every run must reproduce the compiled reference's search
trajectory byte for byte on every rank."""
import multiprocessing as mp
import os
import socket

import pytest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "runs")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, run, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import paper_2004_08140_b200 as gevo
    from paper_2004_08140_b200 import dist as gdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gdist.install_collective()
        bench, seed, pop, gens, mode, train, held = run
        log, rep, st = gevo.run_search(bench, seed, pop, gens, mode, -1.0, train, held, jobs=2)
        q.put((rank, log, rep, st.candidates, st.batches))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,run,world", [
    ("config1_nw-sync", ("nw-sync", 1, 32, 5, "default", 3, 3), 2),
    ("small_hot-memo_mo", ("hot-memo", 3, 16, 4, "mo", 3, 2), 2),
    ("config1_nw-sync", ("nw-sync", 1, 32, 5, "default", 3, 3), 4),
])
def test_sharded_search_matches_reference_trajectory(name, run, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, run, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=600) for _ in procs))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref_log = open(os.path.join(GOLDEN, name, "log.csv")).read()
    ref_rep = open(os.path.join(GOLDEN, name, "report.json")).read()
    for rank in range(world):
        log, rep, cands, batches = res[rank]
        assert log == ref_log, rank
        assert rep.replace('"jobs": 2,', '"jobs": 1,') == ref_rep, rank
        assert cands > 0 and batches > 0


def test_nccl_exchange_search_matches_reference_trajectory():
    """In-library NCCL all-gather of the records (world 1 on this box)."""
    import ctypes
    import sys
    sys.path.insert(0, ROOT)
    import paper_2004_08140_b200 as gevo
    from paper_2004_08140_b200 import lib
    uid = ctypes.create_string_buffer(128)
    assert lib().gevo_nccl_unique_id(uid) == 0, gevo.lib().gevo_last_error()
    assert lib().gevo_set_nccl(0, 1, uid) == 0, gevo.lib().gevo_last_error()
    try:
        log, rep, st = gevo.run_search("nw-sync", 1, 32, 5, "default", -1.0, 3, 3, jobs=2)
    finally:
        lib().gevo_set_nccl(0, 0, None)
    ref = os.path.join(GOLDEN, "config1_nw-sync")
    assert log == open(os.path.join(ref, "log.csv")).read()
    assert rep.replace('"jobs": 2,', '"jobs": 1,') == open(os.path.join(ref, "report.json")).read()
