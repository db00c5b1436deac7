"""Multi-GPU plumbing for the attribution path.

Records are independent (profiles "distributed evenly across the available
ranks"), so each rank attributes a contiguous shard of the stream into its own histogram
and one sum-reduction combines them (accumulators "aggregated by a second
reduction"); on GPUs that is one NCCL reduce of H_inst || U over NVLink.  Integer addition
is associative, so the result is bit-identical for every rank count and shard split.
"""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int, root_less: int = 0) -> tuple[int, int]:
    """Records [floor(r*n/N), floor((r+1)*n/N)) of rank r of N (balanced by records).

    root_less = D > 0: rank 0 also runs the roll-up / CCT / metrics after the reduce, so it
    takes D records fewer than each other rank (D = that analysis time in records of
    attribution time, measured by bench.py): n0 = max(0, floor((n - (N-1) D) / N)) records
    [0, n0) for rank 0, the rest [n0, n) split evenly over ranks 1..N-1.  Any split gives the
    same reduced histogram (integer sums)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} of {world}")
    if root_less <= 0 or world == 1:
        return (n * rank) // world, (n * (rank + 1)) // world
    n0 = max(0, (n - (world - 1) * root_less) // world)
    if rank == 0:
        return 0, n0
    m, k, o = n - n0, rank - 1, world - 1
    return n0 + (m * k) // o, n0 + (m * (k + 1)) // o


def reduce_histogram(hist, dst: int = 0, group=None) -> None:
    """Sum the (int64-viewed u64) histogram buffer of every rank into `dst`, in place.

    `hist` is one contiguous tensor holding H_inst followed by U, so a single collective
    moves the whole payload; NCCL on CUDA tensors, gloo on CPU tensors (tests).  Two's-
    complement int64 sums equal u64 sums bit for bit."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    dist.reduce(hist, dst=dst, op=dist.ReduceOp.SUM, group=group)


def reduce_scatter_histogram(hist, bounds, n_inst: int, group=None) -> None:
    """Reduce-scatter of H_inst || U at function-aligned instruction bounds (gpa_partition_structure):
    rank r receives the element-wise sum of rows [bounds[r], bounds[r+1]) (the last rank also U),
    in place; the rest of its buffer keeps its own partial sums.  One reduce per destination (the
    parts are uneven), so NCCL and gloo run the same code; "aggregated by a second
    reduction", after which each rank generates the statistics of its part."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    world = dist.get_world_size(group)
    assert len(bounds) == world + 1 and bounds[0] == 0 and bounds[-1] == n_inst
    for r in range(world):
        a = int(bounds[r]) * 16
        b = (int(bounds[r + 1]) * 16) if r < world - 1 else hist.numel()
        if b > a:
            dist.reduce(hist[a:b], dst=r, op=dist.ReduceOp.SUM, group=group)


def shard_trace(lines: dict, rank: int, world: int) -> dict:
    """f4: ranks of a trace set are independent problems, so worker r of N takes
    the contiguous range of trace ranks whose change points fall in [floor(r*E/N),
    floor((r+1)*E/N)) by their first change point (balanced by change points; no collective).
    Returns the sub-table (line_off rebased to 0, line_scope rebased to 0) plus scope0 /
    event0 / event1: slice the device event arrays with [event0:event1] and write results
    to rows scope0 .. scope0 + n_scopes of the full outputs."""
    import numpy as np
    lo = np.asarray(lines["line_off"], np.uint64)
    ls = np.asarray(lines["line_scope"], np.uint32)
    S = int(lines["n_scopes"])
    E = int(lo[-1]) if len(lo) else 0
    first = np.searchsorted(ls, np.arange(S + 1), side="left")     # first line of each scope
    scope_start = lo[np.minimum(first, len(lo) - 1)].astype(np.int64)
    a, b = shard_range(E, rank, world)
    s0 = int(np.searchsorted(scope_start[:S], a, side="left")) if rank else 0
    s1 = int(np.searchsorted(scope_start[:S], b, side="left")) if rank < world - 1 else S
    l0, l1 = int(first[s0]), int(first[s1])
    e0, e1 = int(lo[l0]), int(lo[l1])
    return dict(line_off=(lo[l0:l1 + 1] - np.uint64(e0)).astype(np.uint64),
                line_kind=np.asarray(lines["line_kind"], np.uint8)[l0:l1],
                line_scope=(ls[l0:l1] - np.uint32(s0)).astype(np.uint32),
                n_scopes=s1 - s0, n_routines=int(lines["n_routines"]), scope0=s0, event0=e0, event1=e1)
