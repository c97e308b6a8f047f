"""Stripe sharding across ranks: stripes are independent, so rank r of
N owns a contiguous stripe range and there is no collective on the data path.  The
only cross-rank operations are the timing barrier and the max-over-ranks reduction
of the measured time (torch.distributed: NCCL on GPUs, gloo in the CPU tests).
"""


def stripe_range(rank, world, total=None, per_rank=None):
    """Global stripe range [lo, hi) of `rank`.

    Weak scaling (per_rank given): every rank owns per_rank stripes.
    Strong scaling (total given): `total` stripes split as evenly as possible.
    """
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    if per_rank is not None:
        return rank * per_rank, (rank + 1) * per_rank
    if total is None:
        raise ValueError("need total or per_rank")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_over_ranks(value, dist=None, device=None):
    """Max of a float across ranks (identity without torch.distributed)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_throughput(bytes_per_rank, seconds_per_rank):
    """Whole-job throughput: all ranks' bytes / the slowest rank's time."""
    return sum(bytes_per_rank) / max(seconds_per_rank)
