"""Multi-GPU host logic (one process per GPU, torch.distributed).

The dynamic block shards by image with no exchange step (masks, indices and
blocks are per image): each rank runs its own images and the only
collectives are bookkeeping -- the max-over-ranks step time and summed
statistics.  Backend "nccl" on GPUs; the same functions run on "gloo" (CPU) in
the tests.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_ranks():
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(n_total: int, rank: int, world: int):
    """Contiguous image range [start, stop) of `rank` when n_total images are split
    over `world` ranks (strong scaling of a global batch); sizes differ by <= 1."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def _reduce(values, op, device):
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=op)
    return [float(v) for v in t.tolist()]


def max_over_ranks(values, device="cpu"):
    """Element-wise max over ranks (timings: the job is as slow as its slowest rank)."""
    return _reduce(values, dist.ReduceOp.MAX, device)


def sum_over_ranks(values, device="cpu"):
    """Element-wise sum over ranks (active-cell counts, images processed)."""
    return _reduce(values, dist.ReduceOp.SUM, device)


def gather_over_ranks(value: float, device="cpu"):
    """[value of rank 0, value of rank 1, ...] on every rank (per-rank step times:
    per-image activation rates vary, so ranks finish at different times)."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
        dist.all_gather(out, t)
        return [float(o.item()) for o in out]
    return [float(t.item())]


def throughput(images_per_rank: int, world: int, steps: int, max_total_ms: float) -> float:
    """Whole-job images/s of a weak-scaling run: all ranks' images over the slowest rank's time."""
    return images_per_rank * world * steps / (max_total_ms / 1e3)


def exchange_logits(logits_local: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """The network's exchange step: every rank's logits [n_local, classes]
    gathered in rank order into [world * n_local, classes] (all_gather_into_tensor;
    NCCL on GPUs, gloo in the CPU tests).  Single process: a copy."""
    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    if out is None:
        out = torch.empty((world * logits_local.shape[0],) + tuple(logits_local.shape[1:]), dtype=logits_local.dtype,
                          device=logits_local.device)
    if world > 1:
        if logits_local.is_cuda:
            dist.all_gather_into_tensor(out, logits_local)
        else:  # gloo has no all_gather_into_tensor
            parts = [torch.empty_like(logits_local) for _ in range(world)]
            dist.all_gather(parts, logits_local)
            torch.cat(parts, out=out)
    else:
        out.copy_(logits_local)
    return out


def active_counts(counts_local, device="cpu"):
    """Per-block active-cell counts summed over the ranks (int64)."""
    t = torch.tensor([int(c) for c in counts_local], dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t)
    return [int(v) for v in t.tolist()]
