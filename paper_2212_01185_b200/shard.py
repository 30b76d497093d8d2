"""Multi-GPU plumbing: images / independent tiles are partitioned across
ranks (one process per GPU) with no collective on the data path
(SURVEY 8(e)).  The only cross-rank traffic is the timing reduction."""

from __future__ import annotations


def shard_range(n_units: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, equal-count slice [lo, hi) of n_units for `rank` (the
    first n_units % world ranks take one extra unit)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_units, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def weak_seeds(per_rank: int, rank: int) -> range:
    """Weak scaling: every rank codes its own `per_rank` images."""
    return range(rank * per_rank, (rank + 1) * per_rank)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank float over the default process group (identity
    when torch.distributed is not initialised)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_msubpx(subpx_per_rank: float, world: int, max_seconds: float) -> float:
    """Whole-job Msubpixel/s: all ranks' sub-pixels over the slowest rank."""
    return subpx_per_rank * world / max_seconds / 1e6
