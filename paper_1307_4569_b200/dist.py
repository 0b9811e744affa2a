"""Multi-GPU plumbing: one process per GPU, signals sharded, no collective on the data path.

The batch of W independent signals is split contiguously over the ranks (SURVEY.md
§8(e)); every rank builds the same plan from the same window (deterministic, no
broadcast) and transforms its shard.  Collectives appear only off the hot path: a MAX
all-reduce of the per-rank device times and, for validation, a gather of per-rank
results.  Works with the "nccl" backend on GPUs and with "gloo" on CPU (tests).
"""
from __future__ import annotations

import os


def world():
    """(world_size, rank, local_rank) from the torchrun environment (1, 0, 0 if absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str | None = None):
    """Initialise torch.distributed when WORLD_SIZE > 1 (NCCL if CUDA is available, else gloo)."""
    import torch
    import torch.distributed as dist
    ws, rank, local = world()
    # the rank's GPU first: NCCL binds its communicator to the current device
    if torch.cuda.is_available():
        torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    if ws > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NSDGT_DIST_BACKEND=gloo: functional runs of the N > 1 path with several ranks on one
        # GPU (NCCL refuses two ranks on one device); not for timing
        backend = backend or os.environ.get("NSDGT_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        dist.init_process_group(backend=backend)
    return ws, rank, local


def shard(W: int, ws: int, rank: int):
    """Contiguous partition of W signals over ws ranks: rank gets [w0, w1)."""
    if ws < 1 or not 0 <= rank < ws:
        raise ValueError("bad rank / world size")
    return (W * rank) // ws, (W * (rank + 1)) // ws


def _device():
    import torch
    import torch.distributed as dist
    return "cuda" if torch.cuda.is_available() and dist.get_backend() == "nccl" else "cpu"


def allreduce(x: float, op: str = "max") -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "sum": dist.ReduceOp.SUM, "min": dist.ReduceOp.MIN}[op])
    return float(t.item())


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def gather_to_rank0(local, W: int):
    """Gather the per-rank shards c[w0:w1] (torch tensors, same trailing shape) into a full
    (W, ...) tensor on rank 0 (None on the other ranks).  Validation only, off the hot path."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    ws, rank = dist.get_world_size(), dist.get_rank()
    if local.is_complex():  # transported as (re, im) pairs: gloo has no complex dtype
        out = gather_to_rank0(torch.view_as_real(local.contiguous()), W)
        return None if out is None else torch.view_as_complex(out.contiguous())
    dev = local.device if _device() == "cuda" else torch.device("cpu")
    tail = tuple(local.shape[1:])
    chunks = [shard(W, ws, r) for r in range(ws)]
    maxn = max(b - a for a, b in chunks)
    buf = torch.zeros((maxn,) + tail, dtype=local.dtype, device=dev)
    buf[: local.shape[0]] = local.to(dev)
    bufs = [torch.zeros_like(buf) for _ in range(ws)] if rank == 0 else None
    dist.gather(buf, gather_list=bufs, dst=0)
    if rank != 0:
        return None
    return torch.cat([bufs[r][: b - a] for r, (a, b) in enumerate(chunks)], dim=0)
