"""Multi-GPU plumbing for batch-sharded stack execution.

Every image is an independent unit of a stack (pooling windows never cross images; BN /
SCALE parameters are per channel and replicated), so the batch shards across ranks with no
data-path collective.  torch.distributed (NCCL on GPUs, gloo on CPU tests) is used only
after the timed region: max-over-ranks times and per-rank output checksums.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import torch
import torch.distributed as dist


def shard(n_total: int, world: int, rank: int) -> Tuple[int, int]:
    """Images [lo, hi) of `rank` when n_total images are split over `world` ranks
    (contiguous, sizes differ by at most one)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _coll_device(device) -> torch.device:
    """gloo reduces CPU tensors; NCCL needs CUDA tensors."""
    if dist.is_initialized() and dist.get_backend() == "nccl":
        return torch.device(device)
    return torch.device("cpu")


def max_over_ranks(values: Sequence[float], device="cpu") -> List[float]:
    """Element-wise max of a small float vector over all ranks (identity without a group)."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return [float(v) for v in values]
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=_coll_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.cpu()]


def gather_stats(values: Sequence[float], device="cpu") -> List[List[float]]:
    """all_gather of a small per-rank float vector (checksums, times) -> one list per rank."""
    vals = [float(v) for v in values]
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return [vals]
    dev = _coll_device(device)
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [[float(v) for v in o.cpu()] for o in out]


def gather_shards(shard_tensor: torch.Tensor, n_total: int, device="cpu") -> torch.Tensor:
    """Concatenate every rank's output shard (images along dim 0) on every rank -- for
    validation outside the timed region only.  Shards may differ in size by one image."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return shard_tensor
    world = dist.get_world_size()
    dev = _coll_device(device)
    per = [shard(n_total, world, r) for r in range(world)]
    mx = max(hi - lo for lo, hi in per)
    pad = torch.zeros((mx,) + tuple(shard_tensor.shape[1:]), dtype=shard_tensor.dtype, device=dev)
    pad[: shard_tensor.shape[0]] = shard_tensor.to(dev)
    out = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(out, pad)
    return torch.cat([o[: hi - lo] for o, (lo, hi) in zip(out, per)], dim=0)
