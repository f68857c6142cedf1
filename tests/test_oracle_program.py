"""oracle.run_program -- the CPU evaluator behind bench.py's LocPIR CPU baseline -- runs a
loc_pir gate program (reference circuit and the flagged folded form) on encrypted inputs
and decrypts to the plaintext answer."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_19871_b200 import workloads as W


def _tiny_case(K):
    b = W.make_batch(1, 2, 4, 2, seed=8)
    b.x[0] = (b.boxes[1, 0] + b.boxes[1, 1]) // 2
    b.y[0] = (b.boxes[1, 2] + b.boxes[1, 3]) // 2
    lay = W.PoolLayout(b)
    pool = np.zeros((lay.total, K.n + 1), np.uint32)
    s = O.NoiseSampler(9, K.p.alpha_in)
    for slots, vals in ((lay.x, b.x), (lay.y, b.y)):
        for i, bit in enumerate(W._bits_signed(vals, b.l).reshape(-1)):
            pool[slots.reshape(-1)[i]] = O.encrypt_bit(int(bit), K.lwe_key, s)
    bb = W._bits_signed(b.boxes, b.l).reshape(-1)
    pool[lay.bnd.reshape(-1), K.n] = np.where(bb == 1, 0x20000000, 0xE0000000)
    for r in range(b.R):
        for j in range(b.m):
            pool[lay.svc[r, j]] = O.encrypt_bit(int((int(b.payload[r]) >> j) & 1), K.lwe_key, s)
    return b, lay, pool


@pytest.mark.parametrize("kw", [{}, {"folded": True}, {"maj": True}])
def test_lane_batched_program_is_bit_identical(kw):
    """run_program(simd=True) -- the LocPIR CPU baseline's lane-batched path, incl. MUX
    (two rotations per gate), MAJ / XOR3 and ANDNY / ORNY -- leaves the pool bit-identical
    to the scalar FFT-mode evaluation."""
    K = O.TfheKeys(80, 5)
    b, lay, pool = _tiny_case(K)
    ops = W.program_ops(b, lay, True, **kw)
    p1, p2 = pool.copy(), pool.copy()
    O.run_program(K, ops, p1, threads=3)
    O.run_program(K, ops, p2, threads=3, simd=True)
    assert np.array_equal(p1, p2)
    got = sum(O.decrypt_bit(p2[lay.out[0, j]], K.lwe_key) << j for j in range(b.m))
    assert got == int(b.truth()[0])


@pytest.mark.parametrize("folded", [False, True])
def test_run_program_loc_pir_tiny(folded):
    K = O.TfheKeys(80, 5)
    b = W.make_batch(1, 2, 4, 2, seed=8)
    b.x[0] = (b.boxes[1, 0] + b.boxes[1, 1]) // 2
    b.y[0] = (b.boxes[1, 2] + b.boxes[1, 3]) // 2
    lay = W.PoolLayout(b)
    pool = np.zeros((lay.total, K.n + 1), np.uint32)
    s = O.NoiseSampler(9, K.p.alpha_in)
    for slots, vals in ((lay.x, b.x), (lay.y, b.y)):
        for i, bit in enumerate(W._bits_signed(vals, b.l).reshape(-1)):
            pool[slots.reshape(-1)[i]] = O.encrypt_bit(int(bit), K.lwe_key, s)
    bb = W._bits_signed(b.boxes, b.l).reshape(-1)
    pool[lay.bnd.reshape(-1), K.n] = np.where(bb == 1, 0x20000000, 0xE0000000)
    for r in range(b.R):
        for j in range(b.m):
            pool[lay.svc[r, j]] = O.encrypt_bit(int((int(b.payload[r]) >> j) & 1), K.lwe_key, s)
    O.run_program(K, W.program_ops(b, lay, True, folded), pool, threads=8)
    got = sum(O.decrypt_bit(pool[lay.out[0, j]], K.lwe_key) << j for j in range(b.m))
    assert got == int(b.truth()[0])
