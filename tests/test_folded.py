"""Flagged plaintext-boundary mode: the constant-folded loc_pir program
must compute exactly the reference loc_pir function (circuits.hpp:276-324) when the
boundaries are plaintext (dataset.hpp:250-253).  CPU tests interpret the emitted gate
program on plaintext bits; the GPU test runs it encrypted."""
import numpy as np
import pytest

from paper_2407_19871_b200 import _abi
from paper_2407_19871_b200 import workloads as W
from paper_2407_19871_b200.engine import loc_pir_folded_program, loc_pir_program, plan


def interpret(ops, pool):
    """Plaintext semantics of every gate kind in include/locpir_b200.h."""
    f = {
        _abi.AND: lambda a, b, c: a & b, _abi.OR: lambda a, b, c: a | b,
        _abi.XOR: lambda a, b, c: a ^ b, _abi.XNOR: lambda a, b, c: 1 - (a ^ b),
        _abi.NAND: lambda a, b, c: 1 - (a & b), _abi.NOR: lambda a, b, c: 1 - (a | b),
        _abi.MUX: lambda a, b, c: b if a else c, _abi.NOT: lambda a, b, c: 1 - a,
        _abi.COPY: lambda a, b, c: a, _abi.ANDNY: lambda a, b, c: (1 - a) & b,
        _abi.ORNY: lambda a, b, c: (1 - a) | b,
        _abi.MAJ: lambda a, b, c: 1 if a + b + c >= 2 else 0,
        _abi.XOR3: lambda a, b, c: a ^ b ^ c,
    }
    for op in ops:
        if op.kind == _abi.CONST:
            pool[op.out] = 1 if op.in0 else 0
            continue
        g = lambda s: pool[s] if s != _abi.SLOT_NONE else 0
        pool[op.out] = f[op.kind](g(op.in0), g(op.in1), g(op.in2))
    return pool


def run_plain(b, folded, xor_tree=True, maj=False, tree=False):
    lay = W.PoolLayout(b)
    pool = {}
    l, m = b.l, b.m
    for slots, vals in ((lay.x, b.x), (lay.y, b.y)):
        bits = W._bits_signed(vals, l)
        for q in range(b.Q):
            for i in range(l):
                pool[int(slots[q, i])] = int(bits[q, i])
    bb = W._bits_signed(b.boxes, l)
    for r in range(b.R):
        for k in range(4):
            for i in range(l):
                pool[int(lay.bnd[r, k, i])] = int(bb[r, k, i])
        for j in range(m):
            pool[int(lay.svc[r, j])] = int((int(b.payload[r]) >> j) & 1)
    ops = W.program_ops(b, lay, xor_tree, folded, maj, tree)
    interpret(ops, pool)
    out = np.zeros(b.Q, np.uint64)
    for q in range(b.Q):
        out[q] = sum(pool[int(lay.out[q, j])] << j for j in range(m))
    return out, ops


@pytest.mark.parametrize("l", [2, 3, 5])
def test_folded_comparators_exhaustive(l):
    """Every box and every query point of the l-bit grid: folded == truth == unfolded."""
    hi = 1 << l
    boxes = [(a, c) for a in range(hi) for c in range(a + 1, hi)]
    pts = np.arange(hi, dtype=np.uint64)
    for (x1, x2) in boxes[:: max(1, len(boxes) // 40)]:
        b = W.make_batch(len(pts), 1, l, 2, seed=1)
        b.x[:] = pts
        b.y[:] = pts[::-1]
        b.boxes[0] = (x1, x2, 0, hi - 1)
        got, _ = run_plain(b, folded=True)
        assert np.array_equal(got, b.truth()), (x1, x2)


@pytest.mark.parametrize("Q,R,l,m", [(5, 7, 8, 3), (3, 16, 16, 8), (2, 9, 13, 9), (4, 3, 32, 4)])
def test_folded_loc_pir_matches_truth_and_reference_circuit(Q, R, l, m):
    b = W.make_batch(Q, R, l, m, seed=Q * 100 + R)
    for q in range(min(Q, R)):  # land some queries inside boxes, some on edges
        b.x[q] = b.boxes[q, 0] if q % 2 else (b.boxes[q, 0] + b.boxes[q, 1]) // 2
        b.y[q] = (b.boxes[q, 2] + b.boxes[q, 3]) // 2
    got, ops = run_plain(b, folded=True)
    ref, _ = run_plain(b, folded=False)
    assert np.array_equal(got, b.truth())
    assert np.array_equal(ref, b.truth())


@pytest.mark.parametrize("l,m", [(16, 8), (13, 9), (6, 3)])
def test_folded_bootstrap_count_and_depth(l, m):
    """At most 4(l-1) + 3 + 2m bootstraps per region (vs 12l + 2m + 3) and depth no
    deeper than the reference circuit's."""
    b = W.make_batch(2, 6, l, m, seed=5)
    lay = W.PoolLayout(b)
    f = plan(W.program_ops(b, lay, True, True))
    u = plan(W.program_ops(b, lay, True, False))
    assert f["blind_rotations"] <= b.Q * b.R * (4 * (l - 1) + 3 + 2 * m)
    assert u["blind_rotations"] == b.units()
    assert f["levels"] <= u["levels"]


def test_folded_rejects_encrypted_boundaries_and_bad_args():
    b = W.make_batch(1, 2, 32, 4, seed=3, encrypted_bounds=True)
    with pytest.raises(ValueError):
        W.program_ops(b, W.PoolLayout(b), folded=True)
    with pytest.raises(Exception):
        loc_pir_folded_program(1, 2, 8, 3, [0] * 8, [0] * 8, np.zeros(3), [0] * 6, [0] * 3, 0)


def ternary_xor_nodes(R):
    """Bootstraps of the flagged modes' XOR3 / XOR tree over R leaves (circuits.hpp
    emit_xor_root with ternary = true)."""
    nodes = 0
    while R > 1:
        nodes += R // 3 + (R % 3 == 2)
        R = R // 3 + (R % 3 != 0)
    return nodes


@pytest.mark.parametrize("R", [1, 2, 3, 4, 5, 9, 10])
@pytest.mark.parametrize("xor_tree", [0, 1])
def test_flagged_modes_skip_the_enc0_xor(R, xor_tree):
    """Flagged modes drop the bootstrapped XOR with Enc(0) that starts each bit column in
    the reference (circuits.hpp:257-261) and, with the tree, reduce a column with XOR3
    nodes (ceil(log3 R) levels); the plaintext answers are the reference function's."""
    l, m, Q = 6, 3, 3
    b = W.make_batch(Q, R, l, m, seed=40 + R)
    for q in range(min(Q, R)):
        b.x[q] = (b.boxes[q, 0] + b.boxes[q, 1]) // 2
        b.y[q] = (b.boxes[q, 2] + b.boxes[q, 3]) // 2
    lay = W.PoolLayout(b)
    ref = plan(W.program_ops(b, lay, xor_tree, folded=False))
    assert ref["blind_rotations"] == b.units()
    want = Q * m * (ternary_xor_nodes(R) if xor_tree else R - 1)
    for kw in (dict(folded=True), dict(folded=True, tree=True), dict(maj=True), dict(tree=True)):
        ops = W.program_ops(b, lay, xor_tree, **kw)
        xors = sum(1 for o in ops if o.kind in (_abi.XOR, _abi.XOR3))
        assert xors == want, kw
        got, _ = run_plain(b, kw.get("folded", False), xor_tree, kw.get("maj", False),
                           kw.get("tree", False))
        assert np.array_equal(got, b.truth()), kw


def test_ternary_xor_tree_depth():
    """R = 256 boxes (cfg3): 6 XOR levels instead of the binary tree's 8 + 1."""
    b = W.make_batch(1, 256, 4, 1, seed=9)
    lay = W.PoolLayout(b)
    f = plan(W.program_ops(b, lay, True, folded=True))
    r = plan(W.program_ops(b, lay, True, folded=False))
    assert ternary_xor_nodes(256) == 129  # 85 + 29 + 10 + 3 + 1 + 1, six levels
    assert f["blind_rotations"] < r["blind_rotations"]
