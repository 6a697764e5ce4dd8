"""Multi-GPU plumbing: one process per GPU, torch.distributed for the exchange.

SURVEY §8(e): solves and sweep points are independent, so they are partitioned
statically across ranks with no data-path collective (weak scaling).  A single
solve split across ranks exchanges exactly one fixed-size best record per rank
(objective, total slices, m tie key) and every rank applies the same
deterministic lexicographic reduce -- the reference's tie-break
(planner.py:850-854) -- so the answer is independent of the rank count.
"""

from __future__ import annotations

import struct
from typing import Callable, Sequence

NO_CANDIDATE = (0, 0.0, 0, (0, 0, 0, 0))


def block_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of n items owned by rank (sizes differ by <= 1)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def better(a: tuple, b: tuple) -> bool:
    """Is best-record a strictly better than b?  Records are (has, obj, slices, tie)."""
    if not a[0]:
        return False
    if not b[0]:
        return True
    if a[1] != b[1]:
        return a[1] > b[1]
    if a[2] != b[2]:
        return a[2] < b[2]
    return tuple(a[3]) < tuple(b[3])


def combine_best(records: Sequence[tuple]) -> int:
    """Index of the winning record (first index on exact ties: records from
    disjoint shards never tie exactly because their tie keys differ)."""
    win = 0
    for i in range(1, len(records)):
        if better(records[i], records[win]):
            win = i
    return win


def pack_record(rec: tuple) -> list[int]:
    """Fixed 7 x int64 wire format: has, objective bits, slices, tie[4]."""
    has, obj, sl, tie = rec
    bits = struct.unpack("<q", struct.pack("<d", float(obj)))[0]
    return [int(has), bits, int(sl), *[int(t) - (1 << 64) if t >= (1 << 63) else int(t)
                                       for t in tie]]


def unpack_record(words: Sequence[int]) -> tuple:
    has, bits, sl, *tie = (int(w) for w in words)
    obj = struct.unpack("<d", struct.pack("<q", bits))[0]
    return (has, obj, sl, tuple(t + (1 << 64) if t < 0 else t for t in tie))


def all_gather_best(rec: tuple, group=None, device=None) -> list[tuple]:
    """One all-gather of the 56-byte best records (NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    t = torch.tensor(pack_record(rec), dtype=torch.int64, device=device)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [unpack_record(o.tolist()) for o in out]


def sharded_map(items: Sequence, solve: Callable[[Sequence], list], group=None) -> list:
    """Solve a block of ``items`` per rank and gather every result on every rank.

    Used for demand/SLO sweep points and batches of independent plans; the
    gather is result plumbing after the timed work, not a data-path collective.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = block_range(len(items), world, rank)
    local = solve(items[lo:hi])
    if world == 1:
        return list(local)
    parts = [None] * world
    dist.all_gather_object(parts, (lo, list(local)), group=group)
    out: list = [None] * len(items)
    for start, res in parts:
        out[start:start + len(res)] = res
    return out


# ------------------------------------------------- one solve split across GPUs

def _result_better(a, b) -> bool:
    """Reference tie-break between feasible plans (planner.py:850-854):
    objective desc, total slices asc, then the canonical m tuple asc."""
    if a.objective != b.objective:
        return a.objective > b.objective
    if a.config.total_slices != b.config.total_slices:
        return a.config.total_slices < b.config.total_slices
    return a.config.m < b.config.m


def pick_sharded(results: Sequence):
    """Combine the per-shard PlanResults of one solve.

    Each shard evaluated a disjoint block of the mixed-radix candidate space
    (jsv_set_shard) and returned its local argmax; the global argmax is the
    best feasible local result.  When no shard is feasible every rank ran the
    same replicated infeasibility diagnosis, so any result (rank 0's) is the
    answer.
    """
    win = None
    for r in results:
        if r.feasible and (win is None or _result_better(r, win)):
            win = r
    return win if win is not None else results[0]


def plan_sharded(app, profile, request, options=None, group=None, device=None):
    """plan() with the exhaustive Stage-2 sweep split across the ranks of ``group``.

    Stage 1 is replicated (deterministic, microseconds); each rank sweeps prefix
    block [Q*r/W, Q*(r+1)/W) of the candidate space and the local results are
    exchanged with one all-gather, then reduced with the reference tie-break on
    every rank -- the answer does not depend on the rank count.
    """
    import torch.distributed as dist

    from . import _native as N
    from . import planner

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    ctx = N.context(device)
    N.set_shard(ctx, rank, world)
    try:
        local = planner.plan_batch(app, profile, [request], options, device=device)[0]
    finally:
        N.set_shard(ctx, 0, 1)
    if world == 1:
        return local
    parts = [None] * world
    dist.all_gather_object(parts, local, group=group)
    return pick_sharded(parts)
