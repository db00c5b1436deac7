"""Multi-GPU plumbing for the attribution path.

Records are independent (profiles "distributed evenly across the available
ranks"), so each rank attributes a contiguous shard of the stream into its own histogram
and one sum-reduction combines them (accumulators "aggregated by a second
reduction"); on GPUs that is one NCCL reduce of H_inst || U over NVLink.  Integer addition
is associative, so the result is bit-identical for every rank count and shard split.
"""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Records [floor(r*n/N), floor((r+1)*n/N)) of rank r of N (balanced by records)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} of {world}")
    return (n * rank) // world, (n * (rank + 1)) // world


def reduce_histogram(hist, dst: int = 0, group=None) -> None:
    """Sum the (int64-viewed u64) histogram buffer of every rank into `dst`, in place.

    `hist` is one contiguous tensor holding H_inst followed by U, so a single collective
    moves the whole payload; NCCL on CUDA tensors, gloo on CPU tensors (tests).  Two's-
    complement int64 sums equal u64 sums bit for bit."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    dist.reduce(hist, dst=dst, op=dist.ReduceOp.SUM, group=group)
