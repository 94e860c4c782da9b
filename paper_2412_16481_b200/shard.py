"""Scene sharding across GPUs of one node.

Scenes are independent (PSH counters are per batch, bw/bucketing.py:294-296;
stage_forward is single-scene, bw/stage.py:111-113; pooling is per slot), so
the multi-GPU forward needs no data-path collective: rank r takes a
contiguous block of scenes, and the only exchanges are a barrier and the
max-over-ranks of the step time (and, for verification, a gather of per-scene
results).  The helpers work with any torch.distributed backend (NCCL on the
B200 box, gloo in the CPU tests).
"""

import torch
import torch.distributed as dist


def scenes_for_rank(n_scenes: int, world: int, rank: int) -> range:
    """Contiguous block partition: the first n % world ranks get one extra."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    q, r = divmod(n_scenes, world)
    start = rank * q + min(rank, r)
    return range(start, start + q + (1 if rank < r else 0))


def _tensor(x, device):
    return torch.tensor([float(x)], dtype=torch.float64, device=device)


def max_over_ranks(x: float, device="cpu") -> float:
    """Max of a scalar over all ranks (the step-time reduction of bench.py)."""
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = _tensor(x, device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_to_root(obj, world: int, rank: int):
    """Gather picklable per-rank results on rank 0 (list ordered by rank)."""
    if world == 1:
        return [obj]
    out = [None] * world if rank == 0 else None
    dist.gather_object(obj, out, dst=0)
    return out
