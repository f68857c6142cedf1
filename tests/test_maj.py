"""Flagged majority-borrow comparators: a < b = borrow out of a' - b' (sign bits flipped),
borrow_{i+1} = MAJ(NOT a'_i, b'_i, borrow_i) -- one bootstrap per bit, boundaries may be
encrypted (cfg5).  The decrypted loc_pir result must equal the reference circuit's."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_19871_b200 import _abi
from paper_2407_19871_b200 import workloads as W
from paper_2407_19871_b200.engine import plan
from test_folded import run_plain


@pytest.mark.parametrize("l", [2, 3, 5])
def test_maj_comparators_exhaustive(l):
    hi = 1 << l
    pts = np.arange(hi, dtype=np.uint64)
    for x1 in range(hi):
        for x2 in range(x1 + 1, hi, max(1, hi // 6)):
            b = W.make_batch(len(pts), 1, l, 2, seed=1, encrypted_bounds=True)
            b.x[:] = pts
            b.y[:] = pts[::-1]
            b.boxes[0] = (x1, x2, 0, hi - 1)
            got, _ = run_plain(b, folded=False, maj=True)
            assert np.array_equal(got, b.truth()), (x1, x2)


@pytest.mark.parametrize("Q,R,l,m", [(5, 7, 8, 3), (3, 16, 16, 8), (2, 5, 32, 4)])
def test_maj_loc_pir_matches_truth(Q, R, l, m):
    b = W.make_batch(Q, R, l, m, seed=Q * 7 + R, encrypted_bounds=True)
    for q in range(min(Q, R)):
        b.x[q] = b.boxes[q, 1] - 1 if q % 2 else (b.boxes[q, 0] + b.boxes[q, 1]) // 2
        b.y[q] = (b.boxes[q, 2] + b.boxes[q, 3]) // 2
    got, ops = run_plain(b, folded=False, maj=True)
    assert np.array_equal(got, b.truth())


@pytest.mark.parametrize("l,m", [(32, 16), (16, 8)])
def test_maj_unit_count_and_depth(l, m):
    b = W.make_batch(2, 6, l, m, seed=5, encrypted_bounds=True)
    lay = W.PoolLayout(b)
    mj = plan(W.program_ops(b, lay, True, False, True))
    ref = plan(W.program_ops(b, lay, True, False, False))
    # flagged modes: per region 4l comparator + 3 AND + m mask bootstraps; each bit column
    # is a ternary XOR3 tree without the reference's XOR with Enc(0)
    from test_folded import ternary_xor_nodes
    assert mj["blind_rotations"] == b.Q * (b.R * (4 * l + m + 3) + m * ternary_xor_nodes(b.R))
    assert ref["blind_rotations"] == b.units()
    assert mj["levels"] < ref["levels"]


def test_oracle_majority_gate_truth_table():
    K = O.TfheKeys(80, 3)
    s = O.NoiseSampler(4, K.p.alpha_in)
    for a in (0, 1):
        for b in (0, 1):
            for c in (0, 1):
                out = K.gate("maj", K.encrypt(a, s), K.encrypt(b, s), K.encrypt(c, s))
                assert K.decrypt(out) == int(a + b + c >= 2)


@pytest.mark.parametrize("level", [80, 128])
def test_oracle_xor3_gate_truth_table(level):
    """XOR3 = BS(-2 (a + b + c)): odd counts land on +1/4, even on -1/4 (mod 1)."""
    K = O.TfheKeys(level, 3)
    s = O.NoiseSampler(5, K.p.alpha_in)
    for a in (0, 1):
        for b in (0, 1):
            for c in (0, 1):
                out = K.gate("xor3", K.encrypt(a, s), K.encrypt(b, s), K.encrypt(c, s))
                assert K.decrypt(out) == a ^ b ^ c


@pytest.mark.gpu
@pytest.mark.parametrize("level", [80, 128])
def test_maj_gates_bit_exact_and_loc_pir_encrypted(level, okeys80, okeys128):
    from paper_2407_19871_b200 import ClientKeys, Context, TfheParams
    p = TfheParams(level)
    keys = ClientKeys(p, 7)
    ctx = Context(p, 0)
    ctx.upload_keys(keys.bk, keys.ksk)
    ok = okeys80 if level == 80 else okeys128
    rng = np.random.default_rng(level)
    bits = rng.integers(0, 2, (3, 64)).astype(np.uint8)
    cts = [keys.encrypt_bits(bits[i], 50 + i) for i in range(3)]
    ctx.pool_reserve(5 * 64)
    for i in range(3):
        ctx.h2d(64 * i, cts[i])
    # one level of 128 (< #SMs): the latency kernel
    ctx.run([(_abi.MAJ, g, 64 + g, 128 + g, 192 + g) for g in range(64)] +
            [(_abi.XOR3, g, 64 + g, 128 + g, 256 + g) for g in range(64)])
    got = ctx.d2h(192, 64)
    assert list(keys.decrypt_bits(got)) == list((bits.sum(0) >= 2).astype(np.uint8))
    got3 = ctx.d2h(256, 64)
    assert list(keys.decrypt_bits(got3)) == list(bits[0] ^ bits[1] ^ bits[2])
    for g in (0, 63):
        assert np.array_equal(got[g], ok.gate("maj", cts[0][g], cts[1][g], cts[2][g]))
        assert np.array_equal(got3[g], ok.gate("xor3", cts[0][g], cts[1][g], cts[2][g]))
    b = W.make_batch(3, 6, 32, 4, seed=level, encrypted_bounds=True)
    for q in range(3):
        b.x[q] = (b.boxes[q, 0] + b.boxes[q, 1]) // 2
        b.y[q] = (b.boxes[q, 2] + b.boxes[q, 3]) // 2
    lay = W.PoolLayout(b)
    ctx.pool_reserve(lay.total)
    W.load_batch(ctx, keys, b, lay, seed=9)
    ctx.counters_reset()
    prog = W.program(ctx, b, lay, maj=True)
    prog.launch()
    assert np.array_equal(W.read_results(ctx, keys, b, lay), b.truth())
    from test_folded import ternary_xor_nodes
    assert ctx.counters()["bootstrap_units"] == b.Q * (b.R * (4 * 32 + 4 + 3) +
                                                       4 * ternary_xor_nodes(b.R))
    prog.close()
    ctx.close()


def test_three_input_gate_noise_margins():
    """Noise budget of the flagged 3-input gates at the noisier 80-bit set: bootstrapped
    outputs have std sigma; MAJ sums three of them (margin 1/8, std sqrt(3) sigma) and XOR3
    -2x three of them (margin 1/4, std 2 sqrt(3) sigma) -- both >= 15 sigma from a decision
    boundary, as is the reference's 2-input XOR (margin 1/4, 2 sqrt(2) sigma)."""
    K = O.TfheKeys(80, 3)
    s = O.NoiseSampler(4, K.p.alpha_in)
    rng = np.random.default_rng(80)
    G = 240
    A, B = rng.integers(0, 2, G), rng.integers(0, 2, G)
    a = np.stack([K.encrypt(int(x), s) for x in A])
    b = np.stack([K.encrypt(int(x), s) for x in B])
    out = K.gate_batch("nand", a, b, O.FFT, 8)
    n = K.n
    ph = (out[:, n].astype(np.int64) - out[:, :n].astype(np.int64) @ K.lwe_key.astype(np.int64))
    ph = (((ph + 2 ** 31) % 2 ** 32) - 2 ** 31) / 2 ** 32
    sigma = (ph - np.where(1 - (A & B), 0.125, -0.125)).std()
    assert 0.125 / (np.sqrt(3) * sigma) > 15
    assert 0.25 / (2 * np.sqrt(3) * sigma) > 15
