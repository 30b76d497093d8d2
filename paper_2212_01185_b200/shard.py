"""Multi-GPU plumbing: images / independent tiles are partitioned across
devices with no collective on the data path (every image or
tile is its own range-coder stream, /root/reference/pkg/src/lpic/codec.py:178-183).

Two users share this module, so the code that the world-2 gloo test runs is
the code the benchmark runs:

* ``bench.py`` under torchrun (one process per GPU): ``rank_units`` picks the
  rank's images, ``reduce_over_ranks`` takes the max time / summed units over
  the process group (the only cross-rank traffic, outside the timed region),
  ``aggregate_rate`` turns them into the whole-job rate.
* ``codec.encode_batch`` / ``decode_batch(..., devices=[...])`` inside one
  process: ``shard_range`` splits the batch, one host thread per device.
"""

from __future__ import annotations


def shard_range(n_units: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, equal-count slice [lo, hi) of n_units for `rank` (the
    first n_units % world ranks take one extra unit)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if n_units < 0:
        raise ValueError("negative unit count")
    base, extra = divmod(n_units, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def rank_units(n: int, rank: int, world: int, scaling: str) -> tuple[int, int]:
    """Unit indices (image seeds / tile indices) [lo, hi) this rank codes.

    weak:   every rank codes its own n units (seeds rank*n ...), so per-GPU
            work is fixed as the GPU count grows;
    strong: n units in total, split contiguously across the ranks."""
    if scaling == "weak":
        return rank * n, (rank + 1) * n
    if scaling == "strong":
        return shard_range(n, rank, world)
    raise ValueError(f"unknown scaling {scaling!r}")


def reduce_over_ranks(times_s, units: float, device=None) -> tuple[list, float]:
    """(max over ranks of every per-rank time, sum over ranks of `units`).

    Identity when torch.distributed is not initialised.  `device` must be a
    CUDA device under NCCL and None (CPU) under gloo."""
    import torch
    import torch.distributed as dist
    times = [float(t) for t in times_s]
    if not (dist.is_available() and dist.is_initialized()):
        return times, float(units)
    t = torch.tensor(times, dtype=torch.float64, device=device)
    u = torch.tensor([float(units)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return [float(v) for v in t.tolist()], float(u.item())


def max_over_ranks(value: float, device=None) -> float:
    return reduce_over_ranks([value], 0.0, device)[0][0]


def aggregate_rate(units_all_ranks: float, max_seconds: float, scale: float = 1e6) -> float:
    """Whole-job rate (default: millions of units per second): every rank's
    units over the slowest rank's time."""
    if max_seconds <= 0:
        raise ValueError("non-positive time")
    return units_all_ranks / max_seconds / scale


def split_for_devices(n: int, devices: list) -> list:
    """[(device, lo, hi)] contiguous slices of n items, empty slices dropped."""
    out = []
    for r, d in enumerate(devices):
        lo, hi = shard_range(n, r, len(devices))
        if hi > lo:
            out.append((d, lo, hi))
    return out
