"""Population sharding and the fitness exchange step.

One process per GPU. Each (variant, test) execution is independent, so the
only data a rank needs from its peers is the per-variant fitness record of
the population it ranks: rank r evaluates its contiguous shard of the
candidate batch, then every rank all-gathers the fixed-size fitness rows
(cost_mean, error_max, accepted) -- 24 bytes per variant -- and runs the GPU
non-dominated sort (rank_population, src/nsga.cpp:88-106) on the gathered
population. The backend is whatever the process group was created with:
NCCL over NVLink on the GPU box, gloo on CPU tensors in the tests.
"""
from __future__ import annotations

import numpy as np

FIT_COLS = 3  # cost_mean, error_max, accepted


def shard_range(n: int, rank: int, world: int) -> tuple:
    """Contiguous, balanced [begin, end) of n variants for `rank` (the first
    n % world ranks take one extra), so gathered shards concatenate back into
    the batch order."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    q, r = divmod(n, world)
    begin = rank * q + min(rank, r)
    return begin, begin + q + (1 if rank < r else 0)


def fitness_rows(vrec) -> np.ndarray:
    """[n, 3] float64 rows from variant records (gevo_variant_record)."""
    out = np.empty((len(vrec), FIT_COLS), np.float64)
    out[:, 0] = vrec["cost_mean"]
    out[:, 1] = vrec["error_max"]
    out[:, 2] = vrec["accepted"]
    return out


def allgather_fitness(rows: np.ndarray, device=None, group=None) -> np.ndarray:
    """All-gather every rank's [n_r, 3] fitness rows into the global [sum n_r, 3]
    array in rank order (shards may be uneven: counts are exchanged first and
    rows are padded to the largest shard for the collective)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = torch.device("cpu") if device is None else torch.device(device)
    n = torch.tensor([rows.shape[0]], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    m = max(counts) if counts else 0
    local = torch.zeros((m, FIT_COLS), dtype=torch.float64, device=dev)
    if rows.shape[0]:
        local[: rows.shape[0]] = torch.from_numpy(np.ascontiguousarray(rows, np.float64)).to(dev)
    out = torch.empty((world * m, FIT_COLS), dtype=torch.float64, device=dev)
    if m:
        if hasattr(dist, "all_gather_into_tensor") and dev.type == "cuda":
            dist.all_gather_into_tensor(out, local, group=group)
        else:
            parts = list(out.split(m))
            dist.all_gather(parts, local, group=group)
            out = torch.cat(parts)
    host = out.cpu().numpy().reshape(world, m, FIT_COLS)
    return np.concatenate([host[r, : counts[r]] for r in range(world)]) if world else host


def accepted_fitness(gathered: np.ndarray) -> tuple:
    """(cost, error, global index) of the accepted variants of a gathered
    population: the FitnessVectors the search ranks."""
    keep = gathered[:, 2] > 0.5
    idx = np.nonzero(keep)[0]
    return gathered[keep, 0], gathered[keep, 1], idx


# ctypes type of gevo_allgather_fn (include/gevo_b200.h)
_ALLGATHER_FN = None
_installed = []


def install_collective(device=None, group=None):
    """Route the engine's record exchange through torch.distributed: every
    candidate batch of run_search is then sharded by variant across the
    process group's ranks and the 48-byte records are all-gathered (NCCL over
    NVLink when the group is NCCL and `device` a CUDA device, gloo on CPU)."""
    import ctypes

    import torch
    import torch.distributed as dist

    from . import lib, _check

    global _ALLGATHER_FN
    if _ALLGATHER_FN is None:
        _ALLGATHER_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                         ctypes.c_void_p)
    world = dist.get_world_size(group)
    dev = torch.device("cpu") if device is None else torch.device(device)

    def gather(_ctx, send, nbytes, recv):
        src = (ctypes.c_uint8 * nbytes).from_address(send)
        t = torch.frombuffer(bytearray(src), dtype=torch.uint8).to(dev)
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t, group=group)
        flat = torch.cat(out).cpu().numpy()
        ctypes.memmove(recv, flat.ctypes.data, flat.nbytes)

    cb = _ALLGATHER_FN(gather)
    _installed.append(cb)  # keep the trampoline alive
    _check(lib().gevo_set_collective(dist.get_rank(group), world, ctypes.cast(cb, ctypes.c_void_p),
                                     None))


def install_nccl(group=None):
    """In-library exchange: the engine all-gathers its records with its own
    NCCL communicator on the device buffers of each evaluation (one process
    per GPU; rank 0's NCCL unique id is broadcast over `group`)."""
    import ctypes

    import torch.distributed as dist

    from . import lib, _check

    uid = ctypes.create_string_buffer(128)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if rank == 0:
        _check(lib().gevo_nccl_unique_id(uid))
    box = [bytes(uid.raw)]
    dist.broadcast_object_list(box, src=0, group=group)
    ctypes.memmove(uid, box[0], 128)
    _check(lib().gevo_set_nccl(rank, world, uid))


def uninstall_nccl():
    from . import lib, _check
    _check(lib().gevo_set_nccl(0, 0, None))


def uninstall_collective():
    from . import lib, _check
    _check(lib().gevo_set_collective(0, 1, None, None))
