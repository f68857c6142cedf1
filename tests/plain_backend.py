"""Plaintext stand-in for the B200 engine behind paper_2407_19871_b200.dist.ShardedLocPir:
pool slots hold bits, gate programs are interpreted with the gate semantics of
include/locpir_b200.h.  Test infrastructure for the multi-rank host logic (gloo)."""
import numpy as np
import torch

from paper_2407_19871_b200 import _abi
from paper_2407_19871_b200 import workloads as W

_F = {
    _abi.AND: lambda a, b, c: a & b, _abi.OR: lambda a, b, c: a | b,
    _abi.XOR: lambda a, b, c: a ^ b, _abi.XNOR: lambda a, b, c: 1 - (a ^ b),
    _abi.NAND: lambda a, b, c: 1 - (a & b), _abi.NOR: lambda a, b, c: 1 - (a | b),
    _abi.MUX: lambda a, b, c: b if a else c, _abi.NOT: lambda a, b, c: 1 - a,
    _abi.COPY: lambda a, b, c: a, _abi.ANDNY: lambda a, b, c: (1 - a) & b,
    _abi.ORNY: lambda a, b, c: (1 - a) | b,
    _abi.MAJ: lambda a, b, c: 1 if a + b + c >= 2 else 0,
    _abi.XOR3: lambda a, b, c: a ^ b ^ c,
}


def interpret(ops, pool):
    for op in ops:
        k, a, b, c, o = (op.kind, op.in0, op.in1, op.in2, op.out) if not isinstance(op, tuple) else op
        if k == _abi.CONST:
            pool[o] = 1 if a else 0
            continue
        g = lambda s: int(pool[s]) if s != _abi.SLOT_NONE else 0
        pool[o] = _F[k](g(a), g(b), g(c))
    return pool


class _Prog:
    def __init__(self, be, ops):
        self.be, self.ops = be, list(ops)
        self.launches = 0

    def launch(self):
        interpret(self.ops, self.be.pool)
        self.launches += 1

    def close(self):
        pass


class PlainBackend:
    row_words = 1

    def __init__(self):
        self.pool = np.zeros(0, np.int64)

    def reserve(self, slots):
        if slots > self.pool.size:
            self.pool = np.concatenate([self.pool, np.zeros(slots - self.pool.size, np.int64)])

    def load(self, b, lay, seed):
        self.pool[lay.x.reshape(-1)] = W._bits_signed(b.x, b.l).reshape(-1)
        self.pool[lay.y.reshape(-1)] = W._bits_signed(b.y, b.l).reshape(-1)
        self.pool[lay.bnd.reshape(-1)] = W._bits_signed(b.boxes, b.l).reshape(-1)
        sb = (b.payload[:, None] >> np.arange(b.m, dtype=np.uint64)) & 1
        self.pool[lay.svc.reshape(-1)] = sb.reshape(-1).astype(np.int64)

    def program(self, ops):
        return _Prog(self, ops)

    def export(self, first, count):
        return torch.from_numpy(self.pool[first:first + count].astype(np.int32).reshape(-1, 1).copy())

    def import_(self, first, t):
        self.pool[first:first + t.shape[0]] = t.numpy().reshape(-1)

    def read_values(self, first, Q, m):
        bits = self.pool[first:first + Q * m].reshape(Q, m).astype(np.uint64)
        return (bits << np.arange(m, dtype=np.uint64)).sum(axis=1)
