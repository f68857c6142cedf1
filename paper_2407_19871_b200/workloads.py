"""LocPIR query workloads of BASELINE.json (configs 0, 2, 3, 4) on the B200 engine.

Builds seeded synthetic inputs with the configs' shapes, lays them out in the
device pool, emits the batched loc_pir gate program (circuits.hpp:276-324 gate for
gate, csrc/circuits.hpp) and computes the plaintext truth: the XOR of the payloads
of all boxes containing the point (SURVEY.md §0.5 -- boxes may overlap, and that is
exactly what the circuit computes).  Coordinates are 16-bit unsigned values u mapped
to the signed word u - 2^15 (order preserving), or l-bit for cfg5.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _abi

CONFIGS = {
    # name: (security bits, queries, boxes, l, m, encrypted boundaries)
    "cfg1": (80, 1, 1, 16, 8, False),
    "cfg3": (128, 1, 256, 16, 32, False),
    "cfg4": (128, 4096, 16, 16, 8, False),
    "cfg5": (128, 1024, 64, 32, 16, True),
}


@dataclass
class LocPirBatch:
    Q: int
    R: int
    l: int
    m: int
    x: np.ndarray          # [Q] unsigned coordinates
    y: np.ndarray
    boxes: np.ndarray      # [R, 4] (x1, x2, y1, y2) unsigned, x1 < x2, y1 < y2
    payload: np.ndarray    # [R] m-bit service values
    encrypted_bounds: bool

    def truth(self) -> np.ndarray:
        """XOR of the payloads of every box with x1 <= x < x2 and y1 <= y < y2."""
        out = np.zeros(self.Q, np.uint64)
        for q in range(self.Q):
            inside = ((self.boxes[:, 0] <= self.x[q]) & (self.x[q] < self.boxes[:, 1]) &
                      (self.boxes[:, 2] <= self.y[q]) & (self.y[q] < self.boxes[:, 3]))
            v = np.uint64(0)
            for p in self.payload[inside]:
                v ^= np.uint64(p)
            out[q] = v
        return out

    def units(self) -> int:
        return self.Q * self.R * (12 * self.l + 2 * self.m + 3)


def make_batch(Q, R, l, m, seed, encrypted_bounds=False) -> LocPirBatch:
    rng = np.random.default_rng(seed)
    hi = 1 << l
    x = rng.integers(0, hi, Q, dtype=np.uint64)
    y = rng.integers(0, hi, Q, dtype=np.uint64)
    boxes = np.zeros((R, 4), np.uint64)
    for r in range(R):
        for axis in (0, 1):
            a, c = (int(v) for v in rng.integers(0, hi, 2, dtype=np.uint64))
            while a == c:
                c = int(rng.integers(0, hi, dtype=np.uint64))
            boxes[r, 2 * axis], boxes[r, 2 * axis + 1] = min(a, c), max(a, c)
    payload = rng.integers(0, 1 << m, R, dtype=np.uint64)
    return LocPirBatch(Q, R, l, m, x, y, boxes, payload, encrypted_bounds)


def _bits_signed(u: np.ndarray, l: int) -> np.ndarray:
    """u (unsigned l-bit) -> bits of the two's-complement word u - 2^(l-1), LSB first."""
    s = (u.astype(np.int64) - (1 << (l - 1))) & ((1 << l) - 1)
    return ((s[..., None] >> np.arange(l)) & 1).astype(np.uint8)


class PoolLayout:
    """Slot assignment for one batch in the device pool.  chunk: the batch is evaluated
    as programs of at most `chunk` queries that share one scratch region (launched one
    after another on the context stream), so scratch is sized for a chunk, not the
    batch -- every intermediate of a loc_pir program has its own slot, ~7.8K slots
    (19.6 MB) per cfg4 query."""

    def __init__(self, b: LocPirBatch, chunk: int | None = None):
        Q, R, l, m = b.Q, b.R, b.l, b.m
        self.chunk = min(Q, chunk) if chunk else Q
        n = 0
        self.x = n + np.arange(Q * l, dtype=np.uint32).reshape(Q, l); n += Q * l
        self.y = n + np.arange(Q * l, dtype=np.uint32).reshape(Q, l); n += Q * l
        self.bnd = n + np.arange(R * 4 * l, dtype=np.uint32).reshape(R, 4, l); n += R * 4 * l
        self.svc = n + np.arange(R * m, dtype=np.uint32).reshape(R, m); n += R * m
        self.out = n + np.arange(Q * m, dtype=np.uint32).reshape(Q, m); n += Q * m
        self.scratch = n
        self.inputs_end = self.out.min()
        from ._abi import lib
        Qc = max(1, self.chunk)
        self.total = n + max(lib().locpir_b200_loc_pir_scratch(Qc, R, l, m),
                             lib().locpir_b200_loc_pir_folded_scratch(Qc, R, l, m))

    def chunks(self):
        """[q_lo, q_hi) query ranges of the programs."""
        Q = self.x.shape[0]
        c = max(1, self.chunk)
        return [(lo, min(Q, lo + c)) for lo in range(0, Q, c)] if Q else []


def load_batch(ctx, keys, b: LocPirBatch, lay: PoolLayout, seed: int):
    """Client-side encryption of the query words (and boundaries for cfg5), encrypted
    service payloads (the preprocessed service sheet, circuits.hpp:118-146), trivial
    boundary words otherwise (dataset.hpp:250-253); uploads to the pool."""
    l, m = b.l, b.m
    qbits = np.concatenate([_bits_signed(b.x, l).reshape(-1), _bits_signed(b.y, l).reshape(-1)])
    ctx.h2d(int(lay.x.min()), keys.encrypt_bits(qbits, seed))
    bbits = _bits_signed(b.boxes, l).reshape(-1)  # [R, 4, l] order == lay.bnd order
    if b.encrypted_bounds:
        ctx.h2d(int(lay.bnd.min()), keys.encrypt_bits(bbits, seed + 1))
    else:
        ops = [(_abi.CONST, int(bit), 0, 0, int(s)) for bit, s in zip(bbits, lay.bnd.reshape(-1))]
        ctx.run(ops)
    sbits = ((b.payload[:, None] >> np.arange(m, dtype=np.uint64)) & 1).astype(np.uint8)
    ctx.h2d(int(lay.svc.min()), keys.encrypt_bits(sbits.reshape(-1), seed + 2))


def signed_boxes(b: LocPirBatch) -> np.ndarray:
    """[R, 4] signed grid values of the boundaries (the words _bits_signed encodes)."""
    return b.boxes.astype(np.int64) - (1 << (b.l - 1))


def program_ops(b: LocPirBatch, lay: PoolLayout, xor_tree=True, folded=False, maj=False,
                tree=False, q_lo: int = 0, q_hi: int | None = None):
    """The loc_pir gate program of queries [q_lo, q_hi) of the batch (default: all).
    Flagged modes (not the reference gate count): folded=True -- plaintext-boundary
    constant folding (plaintext boundaries only); maj=True --
    majority-borrow comparators; tree=True -- log-depth comparators (latency mode)."""
    from .engine import loc_pir_program_ex
    if folded and b.encrypted_bounds:
        raise ValueError("constant folding needs plaintext boundaries")
    if folded and maj:
        raise ValueError("the majority comparator works on boundary slots, not folded ones")
    q_hi = b.Q if q_hi is None else q_hi
    Q = q_hi - q_lo
    x, y, out = lay.x[q_lo:q_hi], lay.y[q_lo:q_hi], lay.out[q_lo:q_hi]
    cmp = "tree" if tree else "maj" if maj else "reference"
    if folded:
        return loc_pir_program_ex(Q, b.R, b.l, b.m, x, y, lay.svc, out,
                                  lay.scratch, boxes_signed=signed_boxes(b), xor_tree=xor_tree,
                                  comparator=cmp)
    return loc_pir_program_ex(Q, b.R, b.l, b.m, x, y, lay.svc, out, lay.scratch,
                              bnd_slots=lay.bnd, xor_tree=xor_tree, comparator=cmp)


def program(ctx, b: LocPirBatch, lay: PoolLayout, xor_tree=True, folded=False, maj=False,
            tree=False):
    return ctx.program(program_ops(b, lay, xor_tree, folded, maj, tree))


def read_results(ctx, keys, b: LocPirBatch, lay: PoolLayout) -> np.ndarray:
    cts = ctx.d2h(int(lay.out.min()), b.Q * b.m)
    bits = keys.decrypt_bits(cts).reshape(b.Q, b.m).astype(np.uint64)
    return (bits << np.arange(b.m, dtype=np.uint64)).sum(axis=1)


def sub_batch(b: LocPirBatch, q_lo: int, q_hi: int, r_lo: int, r_hi: int) -> LocPirBatch:
    """Queries [q_lo, q_hi) against boxes [r_lo, r_hi) of a batch (multi-GPU shards)."""
    return LocPirBatch(q_hi - q_lo, r_hi - r_lo, b.l, b.m, b.x[q_lo:q_hi].copy(),
                       b.y[q_lo:q_hi].copy(), b.boxes[r_lo:r_hi].copy(),
                       b.payload[r_lo:r_hi].copy(), b.encrypted_bounds)


def combine_ops(G: int, Q: int, m: int, part_first: int, out_first: int, scratch_first: int):
    """Rank-0 combine of G box-shard partials: per query and bit
    column a balanced XOR tree over the G partial roots, then one XOR with Enc(0) -- G
    XOR units, so with the shards' N_g - 1 each the total stays N*m.
    Partial (g, q, j) sits at slot part_first + (g*Q + q)*m + j; output (q, j) at
    out_first + q*m + j.  Uses at most Q*m*G scratch slots from scratch_first."""
    ops = []
    nxt = scratch_first
    for q in range(Q):
        for j in range(m):
            zero = nxt
            nxt += 1
            ops.append((_abi.CONST, 0, _abi.SLOT_NONE, _abi.SLOT_NONE, zero))
            lvl = [part_first + (g * Q + q) * m + j for g in range(G)]
            while len(lvl) > 1:
                nl = []
                for i in range(0, len(lvl) - 1, 2):
                    ops.append((_abi.XOR, lvl[i], lvl[i + 1], _abi.SLOT_NONE, nxt))
                    nl.append(nxt)
                    nxt += 1
                if len(lvl) & 1:
                    nl.append(lvl[-1])
                lvl = nl
            ops.append((_abi.XOR, zero, lvl[0], _abi.SLOT_NONE, out_first + q * m + j))
    return ops
