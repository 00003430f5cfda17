"""Multi-GPU sharding of a Monte Carlo batch: contiguous run-id ranges per rank, no collective on
the hot path, one gather of the per-instance records at the end.

Mirrors how the reference distributes work — independent instances pulled by workers, results
written into slots indexed by run_id so the output is ordered and independent of worker count
(proj/include/ptopt/montecarlo.hpp:137-175).  Here a "worker" is one process per GPU and the
slot order is restored by gathering the ranks' contiguous ranges in rank order.
"""
from __future__ import annotations

import numpy as np


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """[first, first+count) of rank `rank`: ranges are contiguous, ordered by rank, cover
    [0, total) exactly and differ in size by at most one."""
    if total < 0 or world < 1 or not (0 <= rank < world):
        raise ValueError("shard_range: bad arguments")
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def gather_records(local: np.ndarray, total: int, group=None, dst: int = 0):
    """Gathers the ranks' structured record arrays (dtype binding.RECORD_DTYPE or any fixed-size
    dtype) onto rank `dst` in run-id order.  Works on the gloo (CPU tensors) and nccl backends;
    returns the full array on `dst`, None elsewhere.  Without an initialised process group the
    local array is the whole batch."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        assert len(local) == total
        return local
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    item = local.dtype.itemsize
    counts = [shard_range(total, world, r)[1] for r in range(world)]
    assert len(local) == counts[rank], (len(local), counts[rank])
    device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
        else torch.device("cpu")
    # equal-size byte buffers (padded to the largest shard) so a plain all_gather suffices
    width = max(counts) * item
    buf = torch.zeros(width, dtype=torch.uint8)
    raw = np.frombuffer(local.tobytes(), dtype=np.uint8)
    buf[: raw.size] = torch.from_numpy(raw.copy())
    buf = buf.to(device)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    if rank != dst:
        return None
    out = np.empty(total, dtype=local.dtype)
    pos = 0
    for r in range(world):
        n = counts[r]
        out[pos:pos + n] = np.frombuffer(parts[r].cpu().numpy()[: n * item].tobytes(), dtype=local.dtype)
        pos += n
    return out


def max_over_ranks(value: float, group=None) -> float:
    """Multi-GPU timings are reported as the maximum over ranks."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
        else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t[0])


def run_batch_sharded(run_fn, total: int, group=None, dst: int = 0, dtype=None):
    """mc::run_batch over all ranks: rank r solves run ids shard_range(total, world, r) with
    `run_fn(count, first_run_id) -> records` (e.g. ``Solver.run_batch`` bound to this rank's
    GPU) and the records are gathered on `dst` in run-id order.  A rank whose range is empty
    (total < world size) contributes an empty array of `dtype` (default: the run-record dtype)
    without calling `run_fn`."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    first, count = shard_range(total, world, rank)
    if count == 0:
        if dtype is None:
            from .binding import RECORD_DTYPE as dtype
        local = np.empty(0, dtype=dtype)
    else:
        local = run_fn(count, first)
    return gather_records(local, total, group=group, dst=dst)
