"""Multi-GPU plumbing (one process per GPU, torch.distributed over NCCL).

SURVEY.md §8(e): queries / gates are independent, so they are sharded across
ranks with no data-path collective; NCCL is used only to broadcast the
evaluation keys once (BK and KSK in torus form, transformed on each GPU by K0)
and to gather result ciphertexts to rank 0.  The same functions run on the gloo
backend with CPU tensors, which is how the multi-rank logic is tested without GPUs.
"""
from __future__ import annotations

import numpy as np


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Static contiguous partition of [0, total) (the reference's parallel_blocks
    mapping, parallel.hpp:26-34): chunk = ceil(total / world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    chunk = (total + world - 1) // world
    lo = min(total, rank * chunk)
    return lo, min(total, lo + chunk)


def broadcast_keys(params, seed: int, rank: int, device=None):
    """Rank 0 generates the key set; BK and KSK (torus form) are broadcast to all ranks.
    Every rank regenerates only the cheap LWE key (n bits) it needs client-side.

    Returns (client_keys, bk_tensor, ksk_tensor) with tensors on `device`
    (a CUDA device under NCCL, None = CPU under gloo)."""
    import torch
    import torch.distributed as dist

    from .engine import ClientKeys
    bk = torch.empty(params.bk_words(), dtype=torch.int32, device=device)
    ksk = torch.empty(params.ksk_words(), dtype=torch.int32, device=device)
    if rank == 0:
        keys = ClientKeys(params, seed)
        bk.copy_(torch.from_numpy(keys.bk.view(np.int32)))
        ksk.copy_(torch.from_numpy(keys.ksk.view(np.int32)))
    else:
        keys = ClientKeys(params, seed, evaluation_keys=False)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast(bk, src=0)
        dist.broadcast(ksk, src=0)
    return keys, bk, ksk


def max_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_to_root(local: "torch.Tensor", total_rows: int, rank: int, world: int):
    """Gathers row-sharded results (shard_range partition) to rank 0; returns the
    full [total_rows, ...] tensor on rank 0 and None elsewhere."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    chunk = (total_rows + world - 1) // world
    pad = torch.zeros((chunk,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)] if rank == 0 else None
    if dist.get_backend() == "nccl":
        # NCCL has no gather: all_gather then keep rank 0's copy
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad)
    else:
        dist.gather(pad, parts, dst=0)
    if rank != 0:
        return None
    out = []
    for r in range(world):
        lo, hi = shard_range(total_rows, r, world)
        out.append(parts[r][:hi - lo])
    return torch.cat(out, 0)
