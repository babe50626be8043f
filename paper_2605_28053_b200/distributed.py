"""Multi-GPU plumbing for owner-sharded serving (one process per GPU, torch.distributed).

Requests shard by owner: π(o) = placement = rank is part of the compatibility key
κ = (ρ, τ, σ, π) (P:427-428 [§4.3]), so no legal group ever spans GPUs and the
READ/WRITE operators need no collective.  Collectives carry only metadata:
the start-of-run broadcast of the config and owner→rank map, a per-step asynchronous
all_gather of each rank's census / group statistics on a side stream (off the critical
path), the barrier around the timed region, the MAX of per-rank times (the contract's
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


def _dist_on() -> bool:
    return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def broadcast_config(obj, src: int = 0):
    """Start of run: rank `src`'s config / owner→rank map to every rank (pickled, one call)."""
    if not _dist_on():
        return obj
    box = [obj if dist.get_rank() == src else None]
    dist.broadcast_object_list(box, src=src)
    return box[0]


class StatsExchange:
    """Per-step asynchronous all_gather of a small int64 vector per rank (census READ / WRITE,
    groups issued, decode steps).  On NCCL the collective is issued from a side stream, so it
    is ordered after nothing on the compute stream and overlaps the next step; `totals()`
    waits for every outstanding exchange and sums over steps and ranks."""

    def __init__(self, width: int, device=None):
        self.width, self.device = width, device
        self.world = dist.get_world_size() if _dist_on() else 1
        self.side = torch.cuda.Stream(device) if device is not None and device.type == "cuda" else None
        self.pending: list = []
        self.sum = torch.zeros(self.world, width, dtype=torch.int64)

    def post(self, values) -> None:
        row = torch.tensor(list(values), dtype=torch.int64)
        if self.world == 1:
            self.sum[0] += row
            return
        if self.side is not None:
            with torch.cuda.stream(self.side):
                inp = row.to(self.device, non_blocking=False)
                out = torch.empty(self.world * self.width, dtype=torch.int64, device=self.device)
                work = dist.all_gather_into_tensor(out, inp, async_op=True)
        else:
            inp = row
            out = torch.empty(self.world * self.width, dtype=torch.int64)
            work = dist.all_gather_into_tensor(out, inp, async_op=True)
        self.pending.append((work, out))

    def totals(self) -> torch.Tensor:
        """[world][width] sums over every posted step (waits for the outstanding exchanges)."""
        for work, out in self.pending:
            work.wait()
            if self.side is not None:
                self.side.synchronize()
            self.sum += out.view(self.world, self.width).cpu()
        self.pending.clear()
        return self.sum.clone()


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
