"""Flagged latency mode: log-depth (tree) comparators (csrc/circuits.hpp emit_less_tree).
Same decrypted loc_pir result as the reference circuit, with plaintext (folded) or slot
boundaries, and a much shallower program for latency-bound batches (cfg1)."""
import numpy as np
import pytest

from paper_2407_19871_b200 import workloads as W
from paper_2407_19871_b200.engine import plan
from test_folded import interpret


def run_plain(b, folded, tree=True):
    lay = W.PoolLayout(b)
    pool = {}
    for slots, vals in ((lay.x, b.x), (lay.y, b.y)):
        bits = W._bits_signed(vals, b.l)
        for q in range(b.Q):
            for i in range(b.l):
                pool[int(slots[q, i])] = int(bits[q, i])
    bb = W._bits_signed(b.boxes, b.l)
    for r in range(b.R):
        for k in range(4):
            for i in range(b.l):
                pool[int(lay.bnd[r, k, i])] = int(bb[r, k, i])
        for j in range(b.m):
            pool[int(lay.svc[r, j])] = int((int(b.payload[r]) >> j) & 1)
    ops = W.program_ops(b, lay, True, folded, False, tree)
    interpret(ops, pool)
    out = np.array([sum(pool[int(lay.out[q, j])] << j for j in range(b.m)) for q in range(b.Q)],
                   np.uint64)
    return out, ops


@pytest.mark.parametrize("folded", [True, False])
@pytest.mark.parametrize("l", [2, 3, 5])
def test_tree_comparators_exhaustive(l, folded):
    hi = 1 << l
    pts = np.arange(hi, dtype=np.uint64)
    for x1 in range(hi):
        for x2 in range(x1 + 1, hi, max(1, hi // 5)):
            b = W.make_batch(len(pts), 1, l, 2, seed=1, encrypted_bounds=not folded)
            b.x[:] = pts
            b.y[:] = pts[::-1]
            b.boxes[0] = (x1, x2, 0, hi - 1)
            got, _ = run_plain(b, folded)
            assert np.array_equal(got, b.truth()), (x1, x2)


@pytest.mark.parametrize("folded", [True, False])
@pytest.mark.parametrize("Q,R,l,m", [(5, 7, 8, 3), (3, 9, 16, 8), (2, 4, 32, 4), (4, 3, 13, 5)])
def test_tree_loc_pir_matches_truth(Q, R, l, m, folded):
    b = W.make_batch(Q, R, l, m, seed=Q * 11 + R, encrypted_bounds=not folded)
    for q in range(min(Q, R)):
        b.x[q] = b.boxes[q, 0] if q % 2 else (b.boxes[q, 0] + b.boxes[q, 1]) // 2
        b.y[q] = (b.boxes[q, 2] + b.boxes[q, 3]) // 2
    got, _ = run_plain(b, folded)
    assert np.array_equal(got, b.truth())


def test_tree_cuts_cfg1_depth():
    """cfg1 (1 query, 1 box, l = 16, m = 8): the reference circuit is ~l+5 waves deep; the
    folded tree needs log2(16) + 4."""
    b = W.make_batch(1, 1, 16, 8, seed=3)
    lay = W.PoolLayout(b)
    ref = plan(W.program_ops(b, lay))["levels"]
    folded = plan(W.program_ops(b, lay, True, True))["levels"]
    tree = plan(W.program_ops(b, lay, True, True, False, True))["levels"]
    enc_tree = plan(W.program_ops(b, lay, True, False, False, True))["levels"]
    assert tree <= 4 + 4 < folded <= ref
    assert enc_tree <= 5 + 4


@pytest.mark.gpu
@pytest.mark.parametrize("level,folded", [(80, True), (128, False)])
def test_tree_loc_pir_encrypted(level, folded):
    from paper_2407_19871_b200 import ClientKeys, Context, TfheParams
    p = TfheParams(level)
    keys = ClientKeys(p, 7)
    ctx = Context(p, 0)
    ctx.upload_keys(keys.bk, keys.ksk)
    b = W.make_batch(3, 4, 16, 8, seed=level, encrypted_bounds=not folded)
    for q in range(3):
        b.x[q] = (b.boxes[q, 0] + b.boxes[q, 1]) // 2
        b.y[q] = (b.boxes[q, 2] + b.boxes[q, 3]) // 2
    lay = W.PoolLayout(b)
    ctx.pool_reserve(lay.total)
    W.load_batch(ctx, keys, b, lay, seed=9)
    prog = W.program(ctx, b, lay, folded=folded, tree=True)
    prog.launch()
    assert np.array_equal(W.read_results(ctx, keys, b, lay), b.truth())
    prog.close()
    ctx.close()
