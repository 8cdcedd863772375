"""Host-side multi-GPU logic: independent NMPC instances are sharded across ranks
with no collective on the data path; only the timing uses a max-reduction over ranks."""
from __future__ import annotations


def shard(total: int, world: int, rank: int) -> range:
    """Contiguous slice of `total` instances for `rank` (sizes differ by at most one)."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar over all ranks (NCCL on GPUs, gloo on CPU); identity when not distributed."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def per_unit_ms(max_ms: float, steps: int, units_per_step: int) -> float:
    """Whole-job ms per unit (one IPM iteration of one KKT system): max-over-ranks time divided by all
    units every rank processed."""
    return max_ms / (steps * units_per_step)
