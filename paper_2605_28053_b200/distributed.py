"""Multi-GPU plumbing for owner-sharded serving (one process per GPU, torch.distributed).

Requests shard by owner: π(o) = placement = rank is part of the compatibility key
κ = (ρ, τ, σ, π) (P:427-428 [§4.3]), so no legal group ever spans GPUs and the
READ/WRITE operators need no collective.  Collectives carry only metadata: the
barrier around the timed region, the MAX of per-rank times (the contract's
max-over-ranks), and end-of-run gathers of versions / output digests.
Backends: "nccl" on the GPU box, "gloo" for CPU tests (tests/test_distributed_gloo.py).
"""
from __future__ import annotations

import hashlib
import os

import torch
import torch.distributed as dist


def env_rank() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (1 process = 1 GPU)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_streams(n_streams_total: int, world: int, rank: int) -> list[int]:
    """Streams (owners) placed on `rank`: π(o) = o mod world (contiguous blocks are equally
    valid on NVSwitch, where every peer is uniform)."""
    return [s for s in range(n_streams_total) if s % world == rank]


def owner_id(stream: int, base: int = 1000) -> int:
    return base + stream


def max_over_ranks(x: float, device=None) -> float:
    """MAX of a per-rank scalar (timings: the job is as slow as its slowest rank)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_dict(d: dict) -> dict:
    """Union of every rank's {owner: value} (versions, digests); keys must be disjoint."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return dict(d)
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, d)
    out: dict = {}
    for p in parts:
        clash = set(out) & set(p)
        if clash:
            raise RuntimeError(f"owners placed on two ranks: {sorted(clash)[:8]}")
        out.update(p)
    return out


def digest(arrays) -> str:
    """sha256 over the raw bytes of a sequence of numpy arrays / tensors (output digests)."""
    h = hashlib.sha256()
    for a in arrays:
        if isinstance(a, torch.Tensor):
            a = a.detach().cpu().contiguous().view(torch.uint8).numpy()
        h.update(memoryview(a.tobytes() if hasattr(a, "tobytes") else bytes(a)))
    return h.hexdigest()
