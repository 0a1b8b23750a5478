"""Request sharding for batched independent edits (BASELINE config 5).

A single SIGE edit does not split across GPUs (one shared mask
per sparse_forward, graph.cpp:619-901), so multi-GPU throughput comes from
independent requests: request i is served by rank i mod world with its own
ActivationCache resident on that GPU. There is no collective on the data
path; torch.distributed (NCCL on the box, gloo in the CPU tests) only carries
the control plane — per-request latencies and output checksums to rank 0.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import torch
import torch.distributed as dist


def requests_for_rank(n_requests: int, world: int, rank: int) -> list[int]:
    """Round-robin ownership: request i -> rank i mod world."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    return list(range(rank, n_requests, world))


@dataclass
class RequestResult:
    request: int
    rank: int
    ms: float
    checksum: float


def serve(n_requests: int, handler: Callable[[int], tuple[float, float]], world: int | None = None,
          rank: int | None = None) -> list[RequestResult] | None:
    """Run `handler(request) -> (ms, checksum)` for every request this rank owns
    and gather all results on rank 0 (None on the other ranks)."""
    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
        rank = dist.get_rank() if dist.is_initialized() else 0
    mine = [RequestResult(i, rank, *handler(i)) for i in requests_for_rank(n_requests, world, rank)]
    if world == 1 or not dist.is_initialized():
        return mine
    gathered: list = [None] * world if rank == 0 else None
    dist.gather_object(mine, gathered, dst=0)
    if rank != 0:
        return None
    out = [r for part in gathered for r in part]
    out.sort(key=lambda r: r.request)
    return out


def groups_for_rank(n_requests: int, world: int, rank: int, group: int) -> list[list[int]]:
    """This rank's requests (i mod world) in consecutive groups of at most
    `group`: each group is served by one grouped engine (one launch per layer
    for all of its requests, Engine.sparse_forward_grouped)."""
    if group < 1:
        raise ValueError("group size must be >= 1")
    mine = requests_for_rank(n_requests, world, rank)
    return [mine[i:i + group] for i in range(0, len(mine), group)]


def serve_grouped(n_requests: int, group_handler: Callable[[list[int]], Sequence[tuple[float, float]]], group: int,
                  world: int | None = None, rank: int | None = None) -> list[RequestResult] | None:
    """Like serve(), but the handler takes a whole group of this rank's requests
    and returns one (ms, checksum) per request of the group."""
    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
        rank = dist.get_rank() if dist.is_initialized() else 0
    mine: list[RequestResult] = []
    for ids in groups_for_rank(n_requests, world, rank, group):
        res = list(group_handler(ids))
        if len(res) != len(ids):
            raise AssertionError(f"group handler returned {len(res)} results for {len(ids)} requests")
        mine += [RequestResult(i, rank, ms, cs) for i, (ms, cs) in zip(ids, res)]
    if world == 1 or not dist.is_initialized():
        return mine
    gathered: list = [None] * world if rank == 0 else None
    dist.gather_object(mine, gathered, dst=0)
    if rank != 0:
        return None
    out = [r for part in gathered for r in part]
    out.sort(key=lambda r: r.request)
    return out


def max_over_ranks(value: float, device: torch.device | None = None) -> float:
    """Max of a per-rank timing over all ranks (multi-GPU numbers are the
    slowest rank's, never a wall-clock average)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def check_cover(results: Sequence[RequestResult], n_requests: int, world: int) -> None:
    """Every request served exactly once, by its owner."""
    got = [r.request for r in results]
    if sorted(got) != list(range(n_requests)):
        raise AssertionError(f"requests served {got}")
    for r in results:
        if r.rank != r.request % world:
            raise AssertionError(f"request {r.request} served by rank {r.rank}")
