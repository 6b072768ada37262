"""Batch sharder over torch.distributed (one process per GPU).

The beamformer's batch entries (frequency channels x polarizations, PAPER.md:393;
ultrasound frames/ensembles) are independent GEMMs, so the path
partitions with NO data-path collective: every rank runs the same
kernels on its own contiguous slice.  When the batch is smaller than the world
(square / M=32 sweeps, batch 1) the N (samples) dimension is split instead; K is
never split (that would need an fp32/int32 reduction).  NCCL is used only for the
optional output gather and for max-over-ranks timing.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    """This rank's share of a (B, M, N, K) problem."""
    b0: int      # first global batch entry
    nb: int      # number of batch entries
    n0: int      # first sample column
    nn: int      # number of sample columns
    mode: str    # "batch" | "samples" | "replica"


def contiguous_slice(total: int, rank: int, world: int):
    """Balanced contiguous split: the first total % world ranks get one extra element."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def plan_shard(B: int, N: int, rank: int, world: int, align_n: int = 4) -> Shard:
    """Strong-scaling split of one global problem: batch slices when B >= world, else
    sample-column slices (kept multiples of `align_n` so every rank keeps the TMA-store
    epilogue, N % 4 == 0)."""
    if world == 1:
        return Shard(0, B, 0, N, "replica")
    if B >= world:
        b0, nb = contiguous_slice(B, rank, world)
        return Shard(b0, nb, 0, N, "batch")
    units = (N + align_n - 1) // align_n
    u0, nu = contiguous_slice(units, rank, world)
    n0 = u0 * align_n
    nn = max(0, min(N, (u0 + nu) * align_n) - n0)
    return Shard(0, B, n0, nn, "samples")


def gather_outputs(local, group=None):
    """Optional output gather (the only data collective): concatenates the
    per-rank [nb,2,M,N] outputs along the batch dimension on every rank.  Requires equal
    shard sizes (all_gather_into_tensor); returns the local tensor when world == 1."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
        return out
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local.contiguous(), group=group)
    return torch.cat(parts, dim=0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (device-timed numbers are reported as the max)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    if dist.get_backend() != "nccl":
        device = "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    """Sum of a scalar over all ranks (e.g. board energy of every GPU of the job)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    if dist.get_backend() != "nccl":
        device = "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
