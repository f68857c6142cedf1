"""The oracle's restatement of TFHE gate bootstrapping (SURVEY.md §8(a')).

Parity of these internals against TFHE 1.1 is unpinned (the library is absent
from /root/reference); they are anchored on the reference's gate-level
behaviour (truth tables, gate_engine.hpp:196-269) and on internal consistency:
the FP64-FFT external product must equal the exact mod-2^32 product."""
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
import numpy as np
import pytest


def _signed(x):
    return ((np.asarray(x, np.int64) + 2 ** 31) % 2 ** 32) - 2 ** 31


def test_fft_roundtrip_and_tables(oracle):
    W, TW, UT = oracle.fft_tables(1024)
    assert W.shape == (256, 2) and tuple(W[0]) == (1.0, 0.0) and tuple(W[128]) == (-0.0, 1.0)
    for k in range(128):  # W[k + 128] = i * W[k] exactly
        assert W[k + 128][0] == -W[k][1] and W[k + 128][1] == W[k][0]
    assert np.array_equal(UT[:, 0], TW[:, 0]) and np.array_equal(UT[:, 1], -TW[:, 1])
    rng = np.random.default_rng(1)
    a = rng.integers(-2 ** 31, 2 ** 31, 1024).astype(np.int32)
    F = oracle.fft_forward(a) / 512  # the 1/M scale lives in the BK (exact)
    acc = np.zeros(1024, np.uint32)
    oracle.fft_inverse_add(F, acc)
    assert np.array_equal(acc.view(np.int32), a)


def test_forward_is_the_twisted_dft_in_bit_reversed_order(oracle):
    """The absorbed-twist Cooley-Tukey forward computes Z_k = sum_j a_j psi^j W^{jk}
    (a_j = d_j + i d_{j+512}) with Z_k in slot bitrev9(k)."""
    rng = np.random.default_rng(3)
    d = rng.integers(-512, 512, 1024)
    F = oracle.fft_forward(d.astype(np.int32))
    z = F[:, 0] + 1j * F[:, 1]
    a = (d[:512] + 1j * d[512:]) * np.exp(1j * np.pi * np.arange(512) / 1024)
    Z = np.fft.ifft(a) * 512
    brv = [int(format(b, "09b")[::-1], 2) for b in range(512)]
    assert np.max(np.abs(z - Z[brv])) < 1e-9


@pytest.mark.parametrize("level", [80, 128])
def test_fft_product_equals_exact_product(oracle, level, okeys80, okeys128):
    K = okeys80 if level == 80 else okeys128
    rng = np.random.default_rng(level)
    for i in (0, 1, K.n - 1):
        tr = rng.integers(0, 2 ** 32, 2 * K.N, dtype=np.uint64).astype(np.uint32)
        e = K.external_product(i, tr, oracle.EXACT)
        f = K.external_product(i, tr, oracle.FFT)
        assert np.array_equal(e, f)


@pytest.mark.parametrize("level", [80, 128])
def test_fft_margin_on_adversarial_maximum_digits(oracle, level, okeys80, okeys128):
    """the FFT rounding margin on maximum-magnitude gadget digits (every digit
    -Bg/2 or Bg/2 - 1: constant, alternating and random-sign patterns) -- external
    products stay equal to the exact product and the margin stays far below 1/2."""
    K = okeys80 if level == 80 else okeys128
    l, bgbit = (2, 10) if level == 80 else (3, 7)
    half = 1 << (bgbit - 1)
    off = sum(half << (32 - q * bgbit) for q in range(1, l + 1)) + (1 << (31 - l * bgbit))

    def word(d):  # torus word whose l digits all equal d
        return (sum((d + half) << (32 - q * bgbit) for q in range(1, l + 1)) - off) % 2 ** 32

    lo, hi = word(-half), word(half - 1)
    rng = np.random.default_rng(level)
    pats = [np.full(2 * K.N, lo), np.full(2 * K.N, hi),
            np.array([lo if j % 2 else hi for j in range(2 * K.N)])]
    pats += [np.where(rng.integers(0, 2, 2 * K.N) == 1, lo, hi) for _ in range(6)]
    oracle.fft_margin(True)
    for tr in pats:
        tr = np.asarray(tr, np.uint64).astype(np.uint32)
        for i in (0, K.n - 1):
            assert np.array_equal(K.external_product(i, tr, oracle.FFT),
                                  K.external_product(i, tr, oracle.EXACT))
    m = oracle.fft_margin(True)
    assert 0.0 < m < (0.25 if level == 80 else 1.0 / 16), m


def test_full_blind_rotation_fft_equals_exact(oracle, okeys80):
    K = okeys80
    s = oracle.NoiseSampler(5, K.p.alpha_in)
    ct = K.encrypt(1, s)
    assert np.array_equal(K.blind_rotate_acc(ct, mode=oracle.EXACT),
                          K.blind_rotate_acc(ct, mode=oracle.FFT))


def test_decomposition_reconstructs(oracle, okeys128):
    K = okeys128
    p = K.p
    rng = np.random.default_rng(3)
    x = rng.integers(0, 2 ** 32, K.N, dtype=np.uint64).astype(np.uint32)
    rec = np.zeros(K.N, np.int64)
    for lev in range(p.l):
        d = K.decompose(x, lev)
        assert d.min() >= -(1 << (p.bgbit - 1)) and d.max() < (1 << (p.bgbit - 1))
        rec += d.astype(np.int64) << (32 - (lev + 1) * p.bgbit)
    err = _signed(rec - x.astype(np.int64))
    assert np.abs(err).max() <= 1 << (31 - p.l * p.bgbit)


def test_mod_switch(oracle):
    assert oracle.mod_switch(0, 1024) == 0
    assert oracle.mod_switch(0x20000000, 1024) == 256
    assert oracle.mod_switch(0xFFFFFFFF, 1024) == 0  # wraps to 2N == 0
    assert oracle.mod_switch((1 << 20) - 1, 1024) == 0
    assert oracle.mod_switch(1 << 20, 1024) == 1


def test_keyswitch_preserves_phase(oracle, okeys128):
    K = okeys128
    # an N-dim encryption of +1/8 under the TRLWE key, then key switch to the LWE key
    rng = np.random.default_rng(4)
    a = rng.integers(0, 2 ** 32, K.N, dtype=np.uint64).astype(np.uint32)
    body = (int(np.sum(a.astype(np.uint64) * K.trlwe_key)) + 0x20000000) % 2 ** 32
    out = K.keyswitch(np.append(a, np.uint32(body)))
    ph = _signed(K.phase(out)) / 2 ** 32
    assert abs(ph - 0.125) < 1 / 64


@pytest.mark.parametrize("level", [80, 128])
def test_bootstrapped_gate_truth_tables(oracle, level, okeys80, okeys128):
    K = okeys80 if level == 80 else okeys128
    s = oracle.NoiseSampler(21, K.p.alpha_in)
    for kind, fn in [("and", lambda a, b: a & b), ("xor", lambda a, b: a ^ b),
                     ("nand", lambda a, b: 1 - (a & b)), ("xnor", lambda a, b: 1 - (a ^ b))]:
        for a in (0, 1):
            for b in (0, 1):
                out = K.gate(kind, K.encrypt(a, s), K.encrypt(b, s))
                assert K.decrypt(out) == fn(a, b), (kind, a, b)
                ph = _signed(K.phase(out)) / 2 ** 32
                assert abs(abs(ph) - 0.125) < 1 / 16  # acceptance.cpp:377-410 noise bound
    sel = K.encrypt(1, s)
    assert K.decrypt(K.gate("mux", sel, K.encrypt(0, s), K.encrypt(1, s))) == 0
    assert K.decrypt(K.gate("mux", K.encrypt(0, s), K.encrypt(0, s), K.encrypt(1, s))) == 1


def _gate_digest(env_lib):
    import hashlib
    import subprocess
    import sys
    code = ("import sys, numpy as np; sys.path.insert(0, %r); from oracle import oracle as O;"
            "K = O.TfheKeys(128, 7); s = O.NoiseSampler(3, K.p.alpha_in);"
            "a = np.stack([K.encrypt(i & 1, s) for i in range(6)]);"
            "b = np.stack([K.encrypt((i >> 1) & 1, s) for i in range(6)]);"
            "sys.stdout.write(K.gate_batch('nand', a, b, O.FFT, 2).tobytes().hex())") % ROOT
    env = dict(os.environ)
    env.pop("LOCPIR_ORACLE_LIB", None)
    if env_lib:
        env["LOCPIR_ORACLE_LIB"] = env_lib
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=600, check=True)
    return hashlib.sha256(r.stdout.encode()).hexdigest()


def test_avx512_baseline_build_is_bit_identical():
    """bench.py's CPU baseline loads the x86-64-v4 build when the host has AVX-512; it must
    produce the same ciphertexts as the default build (-ffp-contract=off, no fast-math)."""
    v4 = os.path.join(ROOT, "oracle", "build", "liboracle_v4.so")
    if " avx512f" not in open("/proc/cpuinfo").read() or not os.path.exists(v4):
        pytest.skip("no AVX-512 host or no v4 build")
    assert _gate_digest(v4) == _gate_digest(None)


@pytest.mark.parametrize("level", [80, 128])
def test_lane_batched_oracle_is_bit_identical(level):
    """oracle gate_batch_simd (the CPU baseline's fast path: one ciphertext per SIMD lane,
    8 per AVX-512 / 4 per AVX2 vector) reproduces the scalar FFT-mode gates bit for bit,
    including a partial lane group and lanes whose a_i = 0 steps are skipped."""
    from oracle import oracle as O
    K = O.TfheKeys(level, 21)
    s = O.NoiseSampler(22, K.p.alpha_in)
    G = O.simd_lanes() + 3
    rng = np.random.default_rng(level)
    A, B = rng.integers(0, 2, G), rng.integers(0, 2, G)
    a = np.stack([K.encrypt(int(x), s) for x in A])
    b = np.stack([K.encrypt(int(x), s) for x in B])
    a[1, :K.n] = 0  # every mod-switched a_i = 0 for this lane: all of its steps skipped
    for kind in ("and", "or", "xor", "xnor", "nand", "nor"):
        want = K.gate_batch(kind, a, b, O.FFT, 4)
        assert np.array_equal(K.gate_batch_simd(kind, a, b, 3), want), kind
