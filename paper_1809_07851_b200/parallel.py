"""Batch-sharded multi-GPU execution: one process per GPU, each
rank runs the whole four-stage pipeline on its own images and transforms the
kernels locally.  There is NO collective on the data path -- the only
torch.distributed calls are the untimed barrier, the max-over-ranks reduction of
the timing, and (for parity checks) an all_gather of outputs outside the timed
region.  The layer's images are independent units (Eq. 5 has no cross-b term,
P:358-370), so sharding the batch changes no arithmetic."""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def shard_range(B: int, rank: int, world: int) -> tuple[int, int]:
    """Images [lo, hi) owned by ``rank`` when B images are split over ``world`` ranks
    (contiguous, sizes differ by at most one)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world (%d/%d)" % (rank, world))
    if B < 0:
        raise ValueError("negative batch")
    base, rem = divmod(B, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def env_rank_world():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def init(backend: str | None = None):
    """Initialise torch.distributed from the torchrun environment (no-op for world 1)."""
    rank, world, local = env_rank_world()
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def barrier():
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


def max_over_ranks(x: float, device=None) -> float:
    """Max of a scalar over ranks (the timing rule: a multi-GPU step lasts as long as its slowest rank)."""
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    """Sum of a scalar over ranks (whole-job byte counts)."""
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def all_gather_scalar(x: float, device=None) -> list:
    """[x of rank 0, x of rank 1, ...] (per-rank timings for the bench line)."""
    if not (dist.is_available() and dist.is_initialized()):
        return [float(x)]
    world = dist.get_world_size()
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    bufs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(bufs, t)
    return [float(b.item()) for b in bufs]


def gather_batch(local: torch.Tensor, B: int, world: int) -> torch.Tensor:
    """All-gather per-rank output shards [b_lo:b_hi] into the full [B, ...] tensor
    (untimed; parity only).  Shards may differ in size by one image."""
    if world == 1:
        return local
    sizes = [shard_range(B, r, world) for r in range(world)]
    maxb = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((maxb,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return torch.cat([bufs[r][:hi - lo] for r, (lo, hi) in enumerate(sizes)], dim=0)
