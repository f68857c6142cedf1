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


def gather_counts_to_root(local: "torch.Tensor", counts: list, rank: int, world: int):
    """Gathers per-rank row blocks of known sizes `counts[r]` to rank 0 (rows padded to
    max(counts) for the collective); returns the concatenation on rank 0, None elsewhere."""
    import torch.distributed as dist
    if world == 1:
        return local
    mx = max(counts)
    pad = local.new_zeros((mx,) + tuple(local.shape[1:]))
    pad[:local.shape[0]] = local
    parts = [pad.new_empty(pad.shape) for _ in range(world)]
    dist.all_gather(parts, pad)  # NCCL has no gather; gloo takes the same path
    if rank != 0:
        return None
    import torch
    return torch.cat([parts[r][:counts[r]] for r in range(world)], 0)


# ---------------------------------------------------------------------------
# Sharded LocPIR: cfg3 shards BOXES (each rank reduces its boxes to a
# partial XOR root, rank 0 gathers and combines); cfg4/cfg5 shard QUERIES (results
# gathered to rank 0).  The flow is written against a small backend so the same code
# runs on the B200 engine (GpuBackend, NCCL) and, in tests, on a plaintext interpreter
# over gloo.
# ---------------------------------------------------------------------------
class GpuBackend:
    """The B200 engine behind the sharded flow: pool slots hold ciphertext rows.

    staging "device" (NCCL): exported rows are device tensors.  The library enqueues its
    copies and programs on the context's stream while NCCL orders its work after torch's
    current stream, so export() makes the current stream wait for the context stream
    (an event) before the collective reads the tensor, and import_() makes the context
    stream wait for the current stream before it reads what the collective wrote.
    staging "host" (gloo, e.g. several ranks sharing one GPU in tests): rows go through
    host memory with synchronous copies."""

    def __init__(self, ctx, keys, device, staging: str = "device"):
        if staging not in ("device", "host"):
            raise ValueError("staging must be 'device' or 'host'")
        self.ctx, self.keys, self.device, self.staging = ctx, keys, device, staging
        self.row_words = ctx.params.n + 1

    def _ctx_stream(self):
        import torch
        h = self.ctx.stream
        cur = torch.cuda.current_stream(self.device)
        if h == cur.cuda_stream:
            return None, cur
        return torch.cuda.ExternalStream(h, device=self.device), cur

    def reserve(self, slots):
        self.ctx.pool_reserve(slots)

    def load(self, b, lay, seed):
        from .workloads import load_batch
        load_batch(self.ctx, self.keys, b, lay, seed)

    def program(self, ops):
        return self.ctx.program(ops)

    def export(self, first, count):
        import torch
        if self.staging == "host":
            rows = self.ctx.d2h(first, count) if count else np.zeros((0, self.row_words), np.uint32)
            return torch.from_numpy(rows.view(np.int32).copy())
        t = torch.empty((count, self.row_words), dtype=torch.int32, device=self.device)
        if count:
            self.ctx.store_device(first, count, t.data_ptr())
        ext, cur = self._ctx_stream()
        if ext is not None:  # the collective (on `cur`) must see the finished copy
            ev = torch.cuda.Event()
            ev.record(ext)
            cur.wait_event(ev)
        return t

    def import_(self, first, t):
        if not t.shape[0]:
            return
        if self.staging == "host":
            self.ctx.h2d(first, t.cpu().numpy().view(np.uint32))
            return
        import torch
        ext, cur = self._ctx_stream()
        if ext is not None:  # the context stream must see what the collective wrote
            ev = torch.cuda.Event()
            ev.record(cur)
            ext.wait_event(ev)
        self.ctx.load_device(first, t.shape[0], t.data_ptr())
        if ext is not None:  # keep `t` alive until the library's copy has read it
            t.record_stream(ext)

    def read_values(self, first, Q, m):
        bits = self.keys.decrypt_bits(self.ctx.d2h(first, Q * m)).reshape(Q, m).astype(np.uint64)
        return (bits << np.arange(m, dtype=np.uint64)).sum(axis=1)


class ShardedLocPir:
    """One LocPIR batch spread over `world` ranks.  mode "boxes": every rank evaluates all
    queries against its box shard (xor_tree mode 2), rank 0 all-gathers the partial roots
    and runs the combine level (workloads.combine_ops).  mode "queries": every rank
    evaluates its query shard against all boxes; outputs are gathered to rank 0.
    Every rank holds the same seeded batch `b` (inputs are encrypted deterministically)."""

    def __init__(self, backend, b, rank, world, mode, seed, folded=False, maj=False, tree=False,
                 chunk=None):
        """chunk (mode "queries"): evaluate the rank's queries as programs of at most
        `chunk` queries sharing one scratch region (workloads.PoolLayout), launched in
        order on the context stream."""
        from . import workloads as W
        self.be, self.b, self.rank, self.world, self.mode = backend, b, rank, world, mode
        Q, R, m = b.Q, b.R, b.m
        self.prog = self.combine = None
        self.progs = []
        if mode == "boxes":
            self.spans = [shard_range(R, r, world) for r in range(world)]
            self.G = sum(1 for lo, hi in self.spans if hi > lo)
            lo, hi = self.spans[rank]
            self.sub = W.sub_batch(b, 0, Q, lo, hi) if hi > lo else None
            xor_mode = 2 if world > 1 else 1
        elif mode == "queries":
            self.spans = [shard_range(Q, r, world) for r in range(world)]
            lo, hi = self.spans[rank]
            self.sub = W.sub_batch(b, lo, hi, 0, R) if hi > lo else None
            xor_mode = 1
        else:
            raise ValueError("mode must be 'boxes' or 'queries'")
        total = 0
        if self.sub is not None:
            self.lay = W.PoolLayout(self.sub, chunk if mode == "queries" else None)
            total = self.lay.total
        # rank-0 regions: gathered partials / outputs, final outputs, combine scratch
        self.part_first = total
        parts = (self.G * Q * m) if mode == "boxes" else (Q * m)
        self.out_first = self.part_first + parts
        self.comb_first = self.out_first + Q * m
        total = self.comb_first + (Q * m * (self.G + 1) if mode == "boxes" else 0)
        backend.reserve(total)
        if self.sub is not None:
            backend.load(self.sub, self.lay, seed)
            self.progs = [backend.program(W.program_ops(self.sub, self.lay, xor_mode, folded, maj,
                                                        tree, lo, hi))
                          for lo, hi in self.lay.chunks()]
            self.prog = self.progs[0]
        if rank == 0 and mode == "boxes" and world > 1:
            self.combine = backend.program(W.combine_ops(self.G, Q, m, self.part_first,
                                                         self.out_first, self.comb_first))

    def local_rows(self):
        return self.sub.Q * self.sub.m if self.sub is not None else 0

    def launch(self):
        """Local program, then the exchange (all-gather / gather to rank 0) and, for box
        shards, rank 0's combine level."""
        import torch.distributed as dist
        for p in self.progs:
            p.launch()
        if self.world == 1:
            return
        b = self.b
        out0 = int(self.lay.out.min()) if self.sub is not None else 0
        if self.mode == "boxes":
            t = self.be.export(out0, self.local_rows()) if self.sub is not None else \
                self.be.export(0, 0).new_zeros((b.Q * b.m, self.be.row_words))
            parts = [t.new_empty(t.shape) for _ in range(self.world)]
            dist.all_gather(parts, t)
            if self.rank == 0:
                g = 0
                for r, (lo, hi) in enumerate(self.spans):
                    if hi > lo:
                        self.be.import_(self.part_first + g * b.Q * b.m, parts[r])
                        g += 1
                self.combine.launch()
        else:
            t = self.be.export(out0, self.local_rows())
            counts = [(hi - lo) * b.m for lo, hi in self.spans]
            full = gather_counts_to_root(t, counts, self.rank, self.world)
            if self.rank == 0:
                self.be.import_(self.part_first, full)

    def results(self):
        """Rank 0: the XOR-sum value of every query of the batch; None elsewhere."""
        if self.rank != 0:
            return None
        b = self.b
        if self.world == 1:
            return self.be.read_values(int(self.lay.out.min()), b.Q, b.m)
        first = self.out_first if self.mode == "boxes" else self.part_first
        return self.be.read_values(first, b.Q, b.m)

    def prepare(self):
        """Size every program's scratch ahead of the first (timed) launch."""
        for p in self.progs + ([self.combine] if self.combine is not None else []):
            if hasattr(p, "prepare"):
                p.prepare()

    def close(self):
        for p in self.progs + ([self.combine] if self.combine is not None else []):
            p.close()
