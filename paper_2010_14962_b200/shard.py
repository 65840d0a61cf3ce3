"""Multi-GPU slice sharding and the reference's ordered aggregation.

Slices are independent and structurally identical (proj/core/src/cutting.hpp:42-46),
so rank g of G takes the contiguous range [g*n/G, (g+1)*n/G) of ket slice ids,
mirroring run_pool's contiguous batch grid (proj/core/src/executor.cpp:113-136).
Each rank reduces its range to one complex on its device; the only collective is an
all-gather of one complex128 per rank, folded in ascending range order on every rank
like ``aggregate`` (executor.cpp:78-111), so the result is bitwise reproducible for a
fixed world size.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def round_count(jobs: int, workers: int) -> int:
    """round_count (executor.cpp:72-76)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return (jobs + workers - 1) // workers


def shard_range(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous, gap-free split of [0, total) into `world` ranges."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (total * rank) // world, (total * (rank + 1)) // world


def aggregate(partials: Sequence[Tuple[int, int, complex]], total: int) -> complex:
    """aggregate (executor.cpp:78-111): fold (lo, hi, value) in ascending lo after
    checking [0, total) is covered exactly once; input order does not matter."""
    parts: List[Tuple[int, int, complex]] = sorted(partials, key=lambda p: p[0])
    at = 0
    for lo, hi, _ in parts:
        if lo < at:
            raise RuntimeError(f"aggregate overlap: range [{lo},{hi}) rewinds past {at}")
        if lo > at:
            raise RuntimeError(f"aggregate gap: [{at},{lo}) has no result")
        if hi < lo or hi > total:
            raise RuntimeError(f"aggregate range [{lo},{hi}) out of bounds")
        at = hi
    if at != total:
        raise RuntimeError(f"aggregate gap: [{at},{total}) has no result")
    if not parts:
        return 0j
    acc = parts[0][2]
    for p in parts[1:]:
        acc += p[2]
    return acc


def gather_partials(local: complex, lo: int, hi: int, group=None):
    """All-gather (lo, hi, re, im) of every rank (one 32-byte record per rank) over
    torch.distributed (NCCL on GPUs, gloo on CPU); returns the list of partials."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    mine = torch.tensor([float(lo), float(hi), local.real, local.imag], dtype=torch.float64, device=dev)
    world = dist.get_world_size(group)
    bufs = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(bufs, mine, group=group)
    out = []
    for b in bufs:
        v = b.cpu().tolist()
        out.append((int(v[0]), int(v[1]), complex(v[2], v[3])))
    return out
