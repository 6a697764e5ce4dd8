"""Multi-GPU plumbing: one process per GPU, torch.distributed for the exchange.

SURVEY §8(e): solves and sweep points are independent, so they are partitioned
statically across ranks with no data-path collective (weak scaling).  A single
solve split across ranks exchanges exactly one fixed-size best record per rank
(feasible, objective, total slices, the chosen items = the m tie key) in ONE
all-gather, and every rank applies the same deterministic lexicographic reduce
-- the reference's tie-break (planner.py:850-854) -- so the answer is
independent of the rank count.
"""

from __future__ import annotations

import struct
from typing import Callable, Sequence

def block_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of n items owned by rank (sizes differ by <= 1)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


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
#
# Wire record of one shard's local best (int64 words, fixed length 3 + 17 T):
#   [feasible, objective bits, total slices, (n_items[t], items[t][0..15]) per task]
# items are the packed (local key << 16 | count) of the chosen bundle, task-index
# (= task-id) order, so the reference's m tuple (planner.py:262) is recoverable
# and the tie-break (planner.py:850-854) is exact across shards.

def _collective_device(group, device):
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device() if device is None else device)
    return torch.device("cpu")


def plan_record(out, n_tasks: int) -> list[int]:
    """Fixed-size wire record of a jsv_plan_out (see the layout above)."""
    from . import _native as N

    bits = struct.unpack("<q", struct.pack("<d", float(out.objective)))[0]
    words = [int(out.feasible), bits, int(out.total_slices)]
    for t in range(n_tasks):
        n = int(out.n_items[t]) if out.has_config else 0
        words.append(n)
        words.extend(int(out.items[t][k]) if k < n else 0 for k in range(N.MAX_ITEMS))
    return words


def _record_key(words: Sequence[int], n_tasks: int):
    from . import _native as N

    obj = struct.unpack("<d", struct.pack("<q", int(words[1])))[0]
    m = []
    for t in range(n_tasks):
        base = 3 + t * (1 + N.MAX_ITEMS)
        for k in range(int(words[base])):
            w = int(words[base + 1 + k])
            m.append((t, w >> 16, w & 0xFFFF))
    return obj, int(words[2]), tuple(m)


def pick_record(records: Sequence[Sequence[int]], n_tasks: int, feasible_only: bool = False):
    """Rank whose local best is the global answer, or None when no shard is feasible.

    Shards are contiguous blocks of the mixed-radix (= depth-first) candidate
    order, so with ``feasible_only`` the lowest feasible rank holds the first
    feasible leaf; otherwise the reference tie-break: objective desc, total
    slices asc, canonical m asc (a strict prefix is smaller, as for tuples).
    """
    win = None
    best = None
    for r, words in enumerate(records):
        if not int(words[0]):
            continue
        if feasible_only:
            return r
        obj, sl, m = _record_key(words, n_tasks)
        if best is None or obj > best[0] or (obj == best[0] and (sl < best[1] or (
                sl == best[1] and m < best[2]))):
            win, best = r, (obj, sl, m)
    return win


def all_gather_records(words: Sequence[int], group=None, device=None) -> list[list[int]]:
    """ONE all-gather of the fixed-size shard records (NCCL over NVLink on B200s, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = _collective_device(group, device)
    t = torch.tensor(list(words), dtype=torch.int64, device=dev)
    out = torch.empty(world * t.numel(), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(out, t, group=group)
    return out.view(world, t.numel()).cpu().tolist()


def combine_sharded(app, profile, request, lw, local, records, feasible_only: bool = False,
                    options=None, device=None):
    """The global PlanResult on every rank from the gathered shard records.

    No shard feasible: every rank ran the same replicated infeasibility
    diagnosis, so the local result is the answer.  Otherwise the winner's
    assignment is re-derived and validated here (jsv_derive); Stage 1 is
    replicated, so the pool statistics are the local ones.
    """
    import ctypes as C

    from . import _native as N
    from . import planner

    T = len(lw.ids)
    win = pick_record(records, T, feasible_only)
    if win is None:
        # no shard holds a feasible allocation: the whole solve, unsharded, gives the
        # reference's infeasible result with its binding constraint (every rank alike)
        outs, lw, _ = planner.solve_records(app, profile, [request], options, device=device)
        return planner.decode_records((N.PlanOut * 1).from_buffer_copy(outs[0]), app, lw, [request])[0]
    own = plan_record(local, T)
    if list(records[win]) == own:
        return planner.decode_records((N.PlanOut * 1).from_buffer_copy(local), app, lw, [request])[0]
    words = records[win]
    n_items = [int(words[3 + t * (1 + N.MAX_ITEMS)]) for t in range(T)] + [0] * (N.MAX_TASKS - T)
    items = [[0] * N.MAX_ITEMS for _ in range(N.MAX_TASKS)]
    for t in range(T):
        base = 3 + t * (1 + N.MAX_ITEMS)
        items[t][:n_items[t]] = [int(w) for w in words[base + 1:base + 1 + n_items[t]]]
    out = planner.derive_record(app, profile, lw, request, n_items, items)
    for name in ("pool_size", "pool_present", "truncated"):
        C.memmove(C.addressof(out) + getattr(N.PlanOut, name).offset,
                  C.addressof(local) + getattr(N.PlanOut, name).offset,
                  C.sizeof(C.c_int32) * N.MAX_TASKS)
    out.nodes, out.leaves, out.dead = local.nodes, local.leaves, local.dead
    return planner.decode_records((N.PlanOut * 1).from_buffer_copy(out), app, lw, [request])[0]


def plan_sharded(app, profile, request, options=None, group=None, device=None):
    """plan() with the exhaustive Stage-2 sweep split across the ranks of ``group``.

    Stage 1 is replicated (deterministic, sub-millisecond); each rank sweeps
    prefix block [Q*r/W, Q*(r+1)/W) of the candidate space
    (jsv_plan_batch_shard), the fixed-size local best records are exchanged
    with ONE all-gather, and every rank reduces them with the reference
    tie-break and re-derives the winner -- the answer does not depend on the
    rank count (reference planner.py:850-855).
    """
    import torch.distributed as dist

    from . import planner
    from .plan_types import PlannerOptions

    options = options or PlannerOptions()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    outs, lw, _ = planner.solve_records(app, profile, [request], options, device=device,
                                        shard=(rank, world))
    local = outs[0]
    records = [plan_record(local, len(lw.ids))]
    if world > 1:
        records = all_gather_records(records[0], group, device)
    return combine_sharded(app, profile, request, lw, local, records,
                           bool(options.feasible_only), options, device)


def plan_day_sharded(app, profile, trace, slice_budget: int, space, slack: float = 0.05,
                     options=None, group=None, device=None) -> list:
    """workload.plan_day with the trace's bins split into contiguous blocks over the
    ranks of ``group`` (bins are independent plans once the sequential demand
    predictions are made; every rank computes those); the blocks are gathered on
    every rank (result plumbing, not a data-path collective)."""
    import torch.distributed as dist

    from . import workload

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = block_range(len(trace.bins), world, rank)
    local = workload.plan_day(app, profile, trace, slice_budget, space, slack, options, device,
                              part=(lo, hi))
    if world == 1:
        return local
    parts = [None] * world
    dist.all_gather_object(parts, local, group=group)
    return [p for part in parts for p in part]

