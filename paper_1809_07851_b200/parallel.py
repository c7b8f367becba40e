"""Multi-GPU execution, one process per GPU.

Batch-sharded: each rank runs the whole four-stage pipeline on its
own images and transforms the kernels locally.  There is NO collective on the data
path -- the only torch.distributed calls are the untimed barrier, the max-over-ranks
reduction of the timing, and (for parity checks) an all_gather of outputs outside the
timed region.  The layer's images are independent units (Eq. 5 has no cross-b term,
P:358-370), and every per-image quantity (including the F16X3 per-image U scale) is
computed per image, so sharding the batch changes no arithmetic.

Element-sharded (``eshard_forward``): the contraction's E
products are independent; rank j owns elements [e0_j, e1_j) of every
image and only those kernel transforms, with one all-to-all of U and one of X (the
real exchange steps -- NCCL over NVLink on a multi-GPU box)."""
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


def _a2a(out: torch.Tensor, inp: torch.Tensor, out_split, in_split, host_staging: bool):
    """all_to_all_single on byte tensors; host_staging: through CPU copies (gloo)."""
    if host_staging:
        o = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(o, inp.cpu(), list(out_split), list(in_split))
        out.copy_(o)
    else:
        dist.all_to_all_single(out, inp, list(out_split), list(in_split))


def eshard_forward(es, x: torch.Tensor, w: torch.Tensor, out: torch.Tensor, ws: torch.Tensor,
                   bufs: dict | None = None, host_staging: bool = False) -> dict:
    """One element-sharded forward of this rank (``es``: a paper_1809_07851_b200.EShard):
    conv_eshard_forward_a -> all-to-all U + all-gather max|U_b| -> forward_b -> all-to-all X
    -> forward_c.  Returns the exchange buffers (reusable through ``bufs``)."""
    dev = x.device
    if bufs is None:
        bufs = {"u_send": torch.empty(max(1, sum(es.u_send)), dtype=torch.uint8, device=dev),
                "u_recv": torch.empty(max(1, sum(es.u_recv)), dtype=torch.uint8, device=dev),
                "x_send": torch.empty(max(1, sum(es.x_send)), dtype=torch.uint8, device=dev),
                "x_recv": torch.empty(max(1, sum(es.x_recv)), dtype=torch.uint8, device=dev),
                "umax": torch.zeros(max(es.batch), dtype=torch.float32, device=dev),
                "umax_all": torch.zeros(sum(es.batch), dtype=torch.float32, device=dev)}
    es.forward_a(x, w, bufs["u_send"], bufs["umax"], ws)
    world = es.world
    if world > 1:
        _a2a(bufs["u_recv"][:sum(es.u_recv)], bufs["u_send"][:sum(es.u_send)], es.u_recv, es.u_send, host_staging)
        parts = [torch.zeros_like(bufs["umax"]) for _ in range(world)]
        if host_staging:
            cp = [p.cpu() for p in parts]
            dist.all_gather(cp, bufs["umax"].cpu())
            parts = [p.to(dev) for p in cp]
        else:
            dist.all_gather(parts, bufs["umax"])
        bufs["umax_all"].copy_(torch.cat([parts[k][:es.batch[k]] for k in range(world)]))
    else:
        bufs["u_recv"][:sum(es.u_recv)].copy_(bufs["u_send"][:sum(es.u_send)])
        bufs["umax_all"].copy_(bufs["umax"][:es.batch[0]])
    es.forward_b(bufs["u_recv"], bufs["umax_all"], bufs["x_send"], ws)
    if world > 1:
        _a2a(bufs["x_recv"][:sum(es.x_recv)], bufs["x_send"][:sum(es.x_send)], es.x_recv, es.x_send, host_staging)
    else:
        bufs["x_recv"][:sum(es.x_recv)].copy_(bufs["x_send"][:sum(es.x_send)])
    es.forward_c(bufs["x_recv"], out, ws)
    return bufs


def eshard_forward_p2p(es, x: torch.Tensor, w: torch.Tensor, out: torch.Tensor, ws: torch.Tensor,
                       bufs: dict | None = None, host_staging: bool = False) -> dict:
    """Element-sharded forward with the U / X exchange over peer memory instead of a collective
    (conv_eshard_forward_a_peer / _b_peer): every rank's receive buffers are IPC-shared device
    memory mapped into every other rank, each rank copies its packed U (X) straight into the
    owners' buffers, and a stream synchronize + barrier orders the phases.  Only the per-image
    F16X3 maxima (a few bytes) still travel through all_gather.  Same results as
    eshard_forward, bit for bit."""
    import paper_1809_07851_b200 as fc
    dev = x.device
    world, rank = es.world, es.rank
    if bufs is None:
        u, xr = fc.IPCBuffer(sum(es.u_recv)), fc.IPCBuffer(sum(es.x_recv))
        if world > 1:
            handles = [None] * world
            dist.all_gather_object(handles, (u.handle, xr.handle))
        else:
            handles = [(u.handle, xr.handle)]
        up = [u.ptr if k == rank else fc.IPCBuffer.open(handles[k][0]) for k in range(world)]
        xp = [xr.ptr if k == rank else fc.IPCBuffer.open(handles[k][1]) for k in range(world)]
        bufs = {"u_buf": u, "x_buf": xr, "u_peers": up, "x_peers": xp,
                "umax": torch.zeros(max(es.batch), dtype=torch.float32, device=dev),
                "umax_all": torch.zeros(sum(es.batch), dtype=torch.float32, device=dev)}
    stream = torch.cuda.current_stream(dev)
    es.forward_a_peer(x, w, bufs["u_peers"], bufs["umax"], ws)
    if world > 1:
        stream.synchronize()  # this rank's U segments have landed in every peer
        parts = [torch.zeros_like(bufs["umax"]) for _ in range(world)]
        if host_staging:
            cp = [p.cpu() for p in parts]
            dist.all_gather(cp, bufs["umax"].cpu())
            parts = [p.to(dev) for p in cp]
        else:
            dist.all_gather(parts, bufs["umax"])
        bufs["umax_all"].copy_(torch.cat([parts[k][:es.batch[k]] for k in range(world)]))
        dist.barrier()  # ... and every peer's in this rank's buffer
    else:
        bufs["umax_all"].copy_(bufs["umax"][:es.batch[0]])
    es.forward_b_peer(bufs["u_buf"].ptr, bufs["umax_all"], bufs["x_peers"], ws)
    if world > 1:
        stream.synchronize()
        dist.barrier()
    es.forward_c(bufs["x_buf"].ptr, out, ws)
    return bufs


def eshard_release(bufs: dict):
    """Unmap the peers' buffers of eshard_forward_p2p (the own buffers free with `bufs`)."""
    import paper_1809_07851_b200 as fc
    for key, own in (("u_peers", "u_buf"), ("x_peers", "x_buf")):
        for p in bufs.get(key, []):
            if p != bufs[own].ptr:
                fc.IPCBuffer.close(p)
    bufs.clear()
