"""Multi-GPU plumbing for the data-parallel path.

Independent systems shard over ranks (one process per GPU, torch.distributed over NCCL); the
solve has NO collective in its data path.  Collectives appear only around it: a barrier before
timing, a MAX all-reduce of the device-measured step time, and one gather of the per-system
statistics (k, converged) at the end.  Host-side logic is backend-agnostic so the N>1 path is
tested with `gloo` on CPU (tests/test_host_cpu.py::test_two_rank_gloo_sharding).
"""
from __future__ import annotations

import os

import numpy as np

from .batch import shard_range

__all__ = ["init_from_env", "shard_range", "local_systems", "max_over_ranks", "gather_stats"]


def init_from_env(backend: str | None = None):
    """Initialise torch.distributed from torchrun's env (RANK/WORLD_SIZE/MASTER_*); returns
    (rank, world, local_rank).  Single-process runs return (0, 1, 0) without a process group."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        import torch
        if backend is None:
            # SG_DIST_BACKEND=gloo: the multi-process harness on fewer GPUs than ranks (a functional
            # check of the N > 1 path; ranks share a device, so its timings mean nothing)
            backend = os.environ.get("SG_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        if backend == "nccl":
            torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend, rank=rank, world_size=world)
    return rank, world, local


def local_systems(n_per_rank: int, rank: int, world: int, base_seed: int = 0):
    """Weak scaling: rank r owns systems [r*n_per_rank, (r+1)*n_per_rank) of the global batch
    (coefficient seed = system id, rhs seed = system id + 10**6 as the reference CLI)."""
    lo = base_seed + rank * n_per_rank
    ids = list(range(lo, lo + n_per_rank))
    return ids, [i + 10**6 for i in ids]


def _coll_device(device):
    """Collectives run on `device` under NCCL and on the host under gloo."""
    import torch.distributed as dist
    return None if dist.get_backend() == "gloo" else device


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    device = _coll_device(device)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_stats(ks, converged, device=None):
    """All-gather per-system (k, converged) so rank 0 can report the whole job."""
    import torch
    import torch.distributed as dist
    ks = np.asarray(ks, dtype=np.int64)
    cv = np.asarray(converged, dtype=np.int64)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return ks, cv
    world = dist.get_world_size()
    device = _coll_device(device)
    local = torch.tensor(np.stack([ks, cv]), dtype=torch.int64, device=device)
    n = torch.tensor([local.shape[1]], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    m = int(max(s.item() for s in sizes))
    pad = torch.full((2, m), -1, dtype=torch.int64, device=device)
    pad[:, : local.shape[1]] = local
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad)
    allv = torch.cat([o[:, : int(s.item())] for o, s in zip(outs, sizes)], dim=1).cpu().numpy()
    return allv[0], allv[1]
