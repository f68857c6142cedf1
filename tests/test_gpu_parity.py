"""Parity of the B200 path against the CPU oracle and the reference's own pins.

Every test calls through the C ABI (include/locpir_b200.h) via the package's
ctypes binding.  Bars:
  * ciphertexts bit-exact with the oracle (FFT and exact modes agree, see
    test_oracle_tfhe.py), hence pre-KS coefficients within 0 of the exact product;
  * decrypted bits equal to the plaintext function (the reference clear engine)
    for truth tables, comparators and loc_pir (test_gate_engine.cpp,
    test_circuits.cpp, acceptance.cpp);
  * gate counters equal to the reference accounting (gate_engine.hpp:31-77).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GATE_FN = {
    "and": lambda a, b: a & b, "or": lambda a, b: a | b, "xor": lambda a, b: a ^ b,
    "xnor": lambda a, b: 1 - (a ^ b), "nand": lambda a, b: 1 - (a & b),
    "nor": lambda a, b: 1 - (a | b),
}


def _signed(x):
    return ((np.asarray(x, np.int64) + 2 ** 31) % 2 ** 32) - 2 ** 31


@pytest.fixture(scope="module")
def dev():
    from paper_2407_19871_b200 import ClientKeys, Context, TfheParams
    out = {}
    for lvl in (80, 128):
        p = TfheParams(lvl)
        keys = ClientKeys(p, 7)
        ctx = Context(p, 0)
        ctx.upload_keys(keys.bk, keys.ksk)
        out[lvl] = (p, keys, ctx)
    yield out
    for _, _, ctx in out.values():
        ctx.close()


@pytest.mark.parametrize("level", [80, 128])
def test_gates_bit_exact_with_oracle(dev, level, okeys80, okeys128):
    from paper_2407_19871_b200 import _abi
    p, keys, ctx = dev[level]
    ok = okeys80 if level == 80 else okeys128
    bits = np.array([0, 0, 1, 1, 0, 1], np.uint8)
    bits2 = np.array([0, 1, 0, 1, 1, 1], np.uint8)
    a = keys.encrypt_bits(bits, 100 + level)
    b = keys.encrypt_bits(bits2, 200 + level)
    for name, kind in [("and", _abi.AND), ("nand", _abi.NAND), ("xnor", _abi.XNOR)]:
        out = ctx.gate_batch_host(kind, a, b)
        assert list(keys.decrypt_bits(out)) == [GATE_FN[name](x, y) for x, y in zip(bits, bits2)]
        for g in (0, 3):
            assert np.array_equal(out[g], ok.gate(name, a[g], b[g])), (name, g)


def test_mux_bit_exact_with_oracle(dev, okeys128):
    from paper_2407_19871_b200 import _abi
    p, keys, ctx = dev[128]
    s, x, y = (keys.encrypt_bits([v], 300 + i) for i, v in enumerate([1, 0, 1]))
    ctx.pool_reserve(8)
    ctx.h2d(0, np.concatenate([s, x, y]))
    ctx.run([(_abi.MUX, 0, 1, 2, 3), (_abi.MUX, 1, 0, 2, 4)])
    out = ctx.d2h(3, 2)
    assert np.array_equal(out[0], okeys128.gate("mux", s[0], x[0], y[0]))
    assert np.array_equal(out[1], okeys128.gate("mux", x[0], s[0], y[0]))
    assert list(keys.decrypt_bits(out)) == [0, 1]


@pytest.mark.parametrize("level", [80, 128])
def test_wide_mux_level_bit_exact_with_oracle(dev, level, okeys80, okeys128):
    """A level of 300 MUX gates: the 600 blind rotations run on K1 and the 300 combined key
    switches (two N-dim inputs summed, + 1/8) on the tensor-core K2t -- its two-input path.
    Every output decrypts to the MUX truth and 12 sampled rows equal the oracle's gate."""
    from paper_2407_19871_b200 import _abi
    p, keys, ctx = dev[level]
    ok = okeys80 if level == 80 else okeys128
    G = 300
    rng = np.random.default_rng(level + 17)
    S, X, Y = (rng.integers(0, 2, G).astype(np.uint8) for _ in range(3))
    s, x, y = keys.encrypt_bits(S, 41), keys.encrypt_bits(X, 42), keys.encrypt_bits(Y, 43)
    ctx.pool_reserve(4 * G)
    ctx.h2d(0, np.concatenate([s, x, y]))
    ctx.run([(_abi.MUX, g, G + g, 2 * G + g, 3 * G + g) for g in range(G)])
    out = ctx.d2h(3 * G, G)
    assert np.array_equal(keys.decrypt_bits(out), np.where(S == 1, X, Y))
    for g in np.linspace(0, G - 1, 12).astype(int):
        assert np.array_equal(out[g], ok.gate("mux", s[g], x[g], y[g])), g


@pytest.mark.parametrize("level", [80, 128])
def test_truth_tables_many_seeds(dev, level):
    """acceptance.cpp:334-375: every gate, both inputs, many encryption seeds."""
    from paper_2407_19871_b200 import _abi
    p, keys, ctx = dev[level]
    seeds = 100
    A = np.tile([0, 0, 1, 1], seeds).astype(np.uint8)
    B = np.tile([0, 1, 0, 1], seeds).astype(np.uint8)
    S = np.repeat([0, 1], 2 * seeds).astype(np.uint8)
    a = keys.encrypt_bits(A, 1 + level)
    b = keys.encrypt_bits(B, 2 + level)
    s = keys.encrypt_bits(S, 3 + level)
    M = len(A)
    ctx.pool_reserve(20 * M)
    ctx.h2d(0, a)
    ctx.h2d(M, b)
    ctx.h2d(2 * M, s)
    kinds = [("and", _abi.AND), ("or", _abi.OR), ("xor", _abi.XOR), ("xnor", _abi.XNOR),
             ("nand", _abi.NAND), ("nor", _abi.NOR)]
    ops = []
    for k, (_, kind) in enumerate(kinds):
        ops += [(kind, g, M + g, 0, (3 + k) * M + g) for g in range(M)]
    ops += [(_abi.MUX, 2 * M + g, g, M + g, 9 * M + g) for g in range(M)]
    ops += [(_abi.NOT, g, 0, 0, 10 * M + g) for g in range(M)]
    ctx.counters_reset()
    ctx.run(ops)
    for k, (name, _) in enumerate(kinds):
        got = keys.decrypt_bits(ctx.d2h((3 + k) * M, M))
        assert np.array_equal(got, [GATE_FN[name](x, y) for x, y in zip(A, B)]), name
    mux = keys.decrypt_bits(ctx.d2h(9 * M, M))
    assert np.array_equal(mux, np.where(S == 1, A, B))
    nots = keys.decrypt_bits(ctx.d2h(10 * M, M))
    assert np.array_equal(nots, 1 - A)
    c = ctx.counters()
    assert c["and"] == M and c["mux"] == M and c["not"] == M
    assert c["bootstrap_units"] == 6 * M + 2 * M
    # output noise stays far inside the 1/16 decision margin (acceptance.cpp:377-410)
    outs = ctx.d2h(3 * M, 6 * M)
    ph = np.array([_signed(keys.phase(o)) for o in outs]) / 2 ** 32
    assert np.abs(np.abs(ph) - 0.125).max() < 1 / 16


def test_long_xor_chain_stays_decryptable(dev):
    """test_gate_engine.cpp:87-97: 1000 dependent XORs (eager, one gate per program)."""
    from paper_2407_19871_b200 import GateEngine
    p, keys, ctx = dev[128]
    eng = GateEngine(ctx, keys, seed=5)
    eng._next_slot = 0
    acc = eng.encrypt(False)
    one = eng.encrypt(True)
    for _ in range(1000):
        acc = eng.hom_xor(acc, one)
    assert eng.decrypt(acc) is False
    acc = eng.hom_xor(acc, one)
    assert eng.decrypt(acc) is True


def _words(patterns, l):
    return np.array([[(pt >> i) & 1 for i in range(l)] for pt in patterns], np.uint8)


def _signed_of(pattern, l):
    return pattern - (1 << l) if pattern >> (l - 1) else pattern


@pytest.mark.parametrize("l", [2, 3, 4, 5, 6])
def test_comparator_exhaustive(dev, l):
    """acceptance.cpp:113-150: every signed l-bit pair, hom_less and hom_less_equal."""
    from paper_2407_19871_b200 import Context
    _run_comparator_pairs(dev[80], l, [(pa, pb) for pa in range(1 << l) for pb in range(1 << l)],
                          seed=40 + l)


def test_comparator_random_16bit(dev):
    """acceptance.cpp:152-160: 1000 random 16-bit pairs."""
    rng = np.random.default_rng(24)
    pairs = [(int(rng.integers(0, 1 << 16)), int(rng.integers(0, 1 << 16))) for _ in range(1000)]
    _run_comparator_pairs(dev[128], 16, pairs, seed=24)


def _run_comparator_pairs(d, l, pairs, seed):
    from paper_2407_19871_b200 import GateEngine
    from paper_2407_19871_b200.circuits import (CipherWord, FixedPointFormat, hom_less,
                                                hom_less_equal)
    p, keys, ctx = d
    eng = GateEngine(ctx, keys, seed=seed)
    fmt = FixedPointFormat(l - 1, 1)
    A = _words([a for a, _ in pairs], l)
    B = _words([b for _, b in pairs], l)
    ca = eng.encrypt_many(A.reshape(-1))
    cb = eng.encrypt_many(B.reshape(-1))
    lt, le = [], []
    with eng.batch():
        for i in range(len(pairs)):
            wa = CipherWord(ca[i * l:(i + 1) * l], fmt)
            wb = CipherWord(cb[i * l:(i + 1) * l], fmt)
            lt.append(hom_less(wa, wb, eng))
            le.append(hom_less_equal(wa, wb, eng))
    got_lt = eng.decrypt_many(lt)
    got_le = eng.decrypt_many(le)
    for i, (pa, pb) in enumerate(pairs):
        sa, sb = _signed_of(pa, l), _signed_of(pb, l)
        assert got_lt[i] == (sa < sb), (pa, pb)
        assert got_le[i] == (sa <= sb), (pa, pb)


def _encode_regions(eng, spec, fmt, m):
    """spec: list of (x1, x2, y1, y2, service) in grid units -> EncodedRegion (trivial
    boundary words, dataset.hpp:250-253; trivial services, circuits.hpp:150-163)."""
    from paper_2407_19871_b200.circuits import (EncodedRegion, PlainWord, constant_word,
                                                trivial_services)
    out = []
    svc = trivial_services([s[4] for s in spec], m, eng)
    for i, (x1, x2, y1, y2, _) in enumerate(spec):
        w = [constant_word(PlainWord.from_integer(v, fmt), eng) for v in (x1, x2, y1, y2)]
        out.append(EncodedRegion(*w, svc[i], i))
    return out


@pytest.mark.parametrize("tree", [False, True])
def test_loc_pir_reference_regions(dev, tree):
    """test_circuits.cpp:150-213: retrieval, zero outside, half-open edges, counts."""
    from paper_2407_19871_b200 import GateEngine
    from paper_2407_19871_b200.circuits import (FixedPointFormat, PlainWord, decrypt_service,
                                                encrypt_word, loc_pir)
    p, keys, ctx = dev[80]
    fmt = FixedPointFormat(4, 2)
    spec = [(0, 8, 0, 8, 5), (8, 16, 0, 8, 3), (-16, -4, -12, -4, 7)]
    cases = [((5, 2), 5), ((9, 1), 3), ((-10, -6), 7), ((28, 28), 0), ((0, 0), 5), ((8, 0), 3),
             ((16, 0), 0), ((5, 8), 0)]
    eng = GateEngine(ctx, keys, seed=29)
    regions = _encode_regions(eng, spec, fmt, 3)
    ctx.counters_reset()
    outs = []
    with eng.batch():
        for (gx, gy), _ in cases:
            x = encrypt_word(PlainWord.from_integer(gx, fmt), eng)
            y = encrypt_word(PlainWord.from_integer(gy, fmt), eng)
            outs.append(loc_pir(x, y, regions, eng, tree=tree))
    for out, (_, want) in zip(outs, cases):
        assert decrypt_service(out, eng) == want
    c = eng.counters()
    N, l, m = 3, 6, 3
    assert c["xnor"] == len(cases) * N * 4 * l and c["mux"] == len(cases) * N * 4 * l
    assert c["and"] == len(cases) * N * (3 + m) and c["xor"] == len(cases) * N * m
    assert c["bootstrap_units"] == len(cases) * N * (12 * l + 2 * m + 3)


def test_loc_pir_synthetic_matches_reference_golden(dev, golden):
    """bench.hpp:345-384 synthetic cases; retrieved value must equal the reference's."""
    from paper_2407_19871_b200 import GateEngine
    from paper_2407_19871_b200.circuits import (PlainWord, decrypt_service, encrypt_word,
                                                format_for_length, loc_pir)
    p, keys, ctx = dev[80]
    rows = np.array(golden["locpir_synthetic_N_l_m_got_expected_units_xnor_mux_and_xor_not_pred"])
    for N, l, m, got_ref, exp, units, *_ in rows.reshape(-1, 12)[:12]:
        N, l, m = int(N), int(l), int(m)
        fmt = format_for_length(l)
        eng = GateEngine(ctx, keys, seed=1000 + N * 100 + l)
        spec = [(4 * i, 4 * i + 4, 4 * i, 4 * i + 4, (37 * i + 11) & ((1 << m) - 1))
                for i in range(N)]
        regions = _encode_regions(eng, spec, fmt, m)
        pt = PlainWord.from_integer(((N - 1) // 2) * 4 + 2, fmt)
        ctx.counters_reset()
        out = loc_pir(encrypt_word(pt, eng), encrypt_word(pt, eng), regions, eng, tree=True)
        assert decrypt_service(out, eng) == got_ref == exp
        assert eng.counters()["bootstrap_units"] == units


@pytest.mark.parametrize("level", [128, 80])
def test_cfg2_full_size_nand_batch(dev, okeys128, okeys80, level):
    """BASELINE configs[1]: 65,536 NAND -- EVERY output ciphertext bit-exact with the CPU
    oracle (its lane-batched FFT-mode path on all host threads, itself bit-identical to the
    scalar oracle, tests/test_oracle_tfhe.py), and every output decrypts right.  Also at
    the 80-bit set."""
    import os
    from paper_2407_19871_b200 import _abi
    p, keys, ctx = dev[level]
    ok = okeys128 if level == 128 else okeys80
    G = 65536
    rng = np.random.default_rng(2)
    A = rng.integers(0, 2, G).astype(np.uint8)
    B = rng.integers(0, 2, G).astype(np.uint8)
    a = keys.encrypt_bits(A, 77)
    b = keys.encrypt_bits(B, 78)
    out = ctx.gate_batch_host(_abi.NAND, a, b)
    assert np.array_equal(keys.decrypt_bits(out), 1 - (A & B))
    want = ok.gate_batch_simd("nand", a, b, os.cpu_count() or 1)
    bad = np.flatnonzero((out != want).any(axis=1))
    assert bad.size == 0, f"{bad.size} of {G} ciphertexts differ from the oracle, first {bad[:5]}"


def test_errors_map_to_reference_exceptions(dev):
    from paper_2407_19871_b200 import GateEngine, InvalidArgument, _abi
    p, keys, ctx = dev[128]
    e1 = GateEngine(ctx, keys, seed=1)
    e2 = GateEngine(ctx, keys, seed=2)
    a = e1.encrypt(True)
    with pytest.raises(InvalidArgument):
        e2.hom_and(a, a)  # cipher bit belongs to a different engine
    with pytest.raises(InvalidArgument):
        ctx.run([(_abi.AND, 0, 1, 0, ctx.pool_capacity + 5)])


@pytest.mark.parametrize("name,Q,R", [("cfg1", 1, 1), ("cfg3", 1, 64), ("cfg4", 8, 16),
                                       ("cfg5", 1, 4)])
def test_locpir_config_shapes_match_plaintext(dev, name, Q, R):
    """BASELINE.json configs 0/2/3/4 shapes (bounded batch sizes): the decrypted loc_pir
    result equals the XOR of the payloads of all boxes containing the point, incl. the
    encrypted-boundary l = 32 variant."""
    from paper_2407_19871_b200 import workloads as W
    sec, _, _, l, m, enc = W.CONFIGS[name]
    p, keys, ctx = dev[sec]
    b = W.make_batch(Q, R, l, m, seed=99 + R, encrypted_bounds=enc)
    # make sure some queries land inside boxes: put query 0 at the centre of box 0
    b.x[0] = (b.boxes[0, 0] + b.boxes[0, 1]) // 2
    b.y[0] = (b.boxes[0, 2] + b.boxes[0, 3]) // 2
    lay = W.PoolLayout(b)
    ctx.pool_reserve(lay.total)
    W.load_batch(ctx, keys, b, lay, seed=7)
    ctx.counters_reset()
    prog = W.program(ctx, b, lay)
    prog.launch()
    got = W.read_results(ctx, keys, b, lay)
    assert np.array_equal(got, b.truth())
    assert ctx.counters()["bootstrap_units"] == b.units()
    prog.close()


def _exact_many(ok, lwe, oracle):
    """EXACT-mode (schoolbook mod 2^32) oracle blind rotations on all host threads
    (ctypes releases the GIL)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
        return list(ex.map(lambda row: ok.blind_rotate_extract(row, mode=oracle.EXACT), lwe))


@pytest.mark.parametrize("level", [80, 128])
@pytest.mark.parametrize("count", [3, 600])  # latency kernel (< SMs) and throughput kernel
def test_pre_keyswitch_coefficients_equal_exact_oracle(dev, level, count, okeys80, okeys128,
                                                       oracle):
    """SURVEY §8(c) parity ladder: the N-dim extracted coefficients (before key switching)
    equal the EXACT mod-2^32 schoolbook oracle -- stated FFT error bound 0 -- on 64
    ciphertexts per case (all 3 of the latency batch), and equal the oracle's FFT mode
    (the same FP64 operations) on every ciphertext of the batch."""
    p, keys, ctx = dev[level]
    ok = okeys80 if level == 80 else okeys128
    rng = np.random.default_rng(level + count)
    lwe = rng.integers(0, 2 ** 32, (count, p.n + 1), dtype=np.uint64).astype(np.uint32)
    got = ctx.debug_blind_rotate(lwe)
    idx = np.unique(np.linspace(0, count - 1, min(count, 64)).astype(int))
    exact = _exact_many(ok, lwe[idx], oracle)
    for g, e in zip(idx, exact):
        assert np.array_equal(got[g], e), g
    for g in range(count):
        assert np.array_equal(got[g], ok.blind_rotate_extract(lwe[g], mode=oracle.FFT)), g


@pytest.mark.parametrize("level", [80, 128])
@pytest.mark.parametrize("count", [191, 192, 1183, 4097])
def test_tensor_core_keyswitch_matches_k2_and_oracle(dev, level, count, okeys80, okeys128,
                                                     monkeypatch):
    """K2t (ks_tc.cuh: the key switch as an INT8 tcgen05 contraction) is bit-exact with K2
    (a context created with LOCPIR_B200_KSTC=0) on EVERY row and with the oracle on sampled
    rows.  K2t takes levels of >= 192 ciphertexts: 191 stays on the split K2s in both
    contexts, 192 is the first K2t level (against K2s), 1183 / 4097 run against the
    CUDA-core K2, 4097 leaves a ragged last M tile.  Rows 0..3 pin the digit extremes: all
    digits 0, all digits 3 (the largest byte sums the int32 accumulators see), and the
    rounding boundary 2^15 - 1 / 2^15 of the digit decomposition."""
    from paper_2407_19871_b200 import Context
    p, keys, ctx = dev[level]
    ok = okeys80 if level == 80 else okeys128
    rng = np.random.default_rng(level * 7 + count)
    lweN = rng.integers(0, 2 ** 32, (count, p.N + 1), dtype=np.uint64).astype(np.uint32)
    lweN[0, :p.N] = 0
    lweN[1, :p.N] = 0xFFFF0000
    lweN[2, :p.N] = 0x7FFF
    lweN[3, :p.N] = 0x8000
    got = ctx.debug_keyswitch(lweN)
    monkeypatch.setenv("LOCPIR_B200_KSTC", "0")
    k2 = Context(p, 0)
    try:
        k2.upload_keys(keys.bk, keys.ksk)
        want = k2.debug_keyswitch(lweN)
    finally:
        k2.close()
    assert np.array_equal(got, want)
    idx = sorted(set(range(4)) | set(np.linspace(0, count - 1, 24).astype(int).tolist()))
    for g in idx:
        assert np.array_equal(got[g], ok.keyswitch(lweN[g])), g


@pytest.mark.parametrize("count", [5, 3000])  # split (small-level) and batched key switch
def test_keyswitch_bit_exact_on_identical_inputs(dev, count, okeys128):
    """K2 bit-exact against the oracle on identical N-dim inputs."""
    p, keys, ctx = dev[128]
    rng = np.random.default_rng(count)
    lweN = rng.integers(0, 2 ** 32, (count, p.N + 1), dtype=np.uint64).astype(np.uint32)
    got = ctx.debug_keyswitch(lweN)
    for g in (0, count // 2, count - 1):
        assert np.array_equal(got[g], okeys128.keyswitch(lweN[g]))


@pytest.mark.parametrize("level", [80, 128])
def test_city_table_end_to_end_matches_reference(dev, golden, level):
    """acceptance.cpp:180-237: the 9-city KDCA table, interior point of every box returns
    its service and an open-sea point returns 0 -- expected values produced by the
    reference itself (tests/golden/ref_vectors.json, city_*), boundaries as trivial words
    (dataset.hpp:250-253), services and queries encrypted."""
    from paper_2407_19871_b200 import GateEngine
    from paper_2407_19871_b200.circuits import (CipherWord, EncodedRegion, FixedPointFormat,
                                                PlainWord, ServiceCiphertext, constant_word,
                                                decrypt_service, encrypt_word, loc_pir)
    p, keys, ctx = dev[level]
    fmt = FixedPointFormat(9, 7)
    m = golden["city_service_bits"][0]
    boxes = np.array(golden["city_boxes_grid_x1_x2_y1_y2_int32"], np.uint32).view(np.int32)
    boxes = boxes.reshape(-1, 4)
    eng = GateEngine(ctx, keys, seed=31)
    eng._next_slot = 0
    regions = []
    for i, (x1, x2, y1, y2) in enumerate(boxes):
        w = [constant_word(PlainWord.from_integer(int(v), fmt), eng) for v in (x1, x2, y1, y2)]
        svc = golden["city_services"][i]
        bits = eng.encrypt_many([(svc >> j) & 1 for j in range(m)])
        regions.append(EncodedRegion(*w, ServiceCiphertext(bits), i))
    q = np.array(golden["city_queries_grid_xy_int32"], np.uint32).view(np.int32).reshape(-1, 2)
    outs = []
    with eng.batch():
        for gx, gy in q:
            x = encrypt_word(PlainWord.from_integer(int(gx), fmt), eng)
            y = encrypt_word(PlainWord.from_integer(int(gy), fmt), eng)
            outs.append(loc_pir(x, y, regions, eng, tree=True))
    got = [decrypt_service(o, eng) for o in outs]
    assert got == golden["city_expected"]


@pytest.mark.parametrize("level", [80, 128])
def test_output_noise_over_1e5_gates(dev, level):
    """acceptance.cpp:377-410: over 10^5 bootstrapped gates every output phase lies within
    1/16 of its nominal +-1/8 (here the real bootstrap replaces the refresh stand-in)."""
    from paper_2407_19871_b200 import _abi
    p, keys, ctx = dev[level]
    G = 100_000
    rng = np.random.default_rng(level)
    A = rng.integers(0, 2, G).astype(np.uint8)
    B = rng.integers(0, 2, G).astype(np.uint8)
    a = keys.encrypt_bits(A, 500 + level)
    b = keys.encrypt_bits(B, 600 + level)
    out = ctx.gate_batch_host(_abi.XOR, a, b)   # XOR doubles input noise: the hardest form
    assert np.array_equal(keys.decrypt_bits(out), A ^ B)
    n = p.n
    ph = (out[:, n].astype(np.int64) - (out[:, :n].astype(np.int64) @ keys.lwe_key.astype(np.int64)))
    ph = (((ph + 2 ** 31) % 2 ** 32) - 2 ** 31) / 2 ** 32
    err = np.abs(ph - np.where(A ^ B, 0.125, -0.125))
    assert err.max() < 1 / 16


def _random_program(rng, n_inputs, n_ops, first_slot):
    """Random SSA gate DAG over n_inputs input slots; returns (ops, plaintext evaluator)."""
    from paper_2407_19871_b200 import _abi
    kinds = [_abi.AND, _abi.OR, _abi.XOR, _abi.XNOR, _abi.NAND, _abi.NOR, _abi.MUX, _abi.NOT,
             _abi.COPY, _abi.CONST, _abi.ANDNY, _abi.ORNY, _abi.MAJ, _abi.XOR3]
    live = list(range(n_inputs))
    ops = []
    nxt = first_slot
    for _ in range(n_ops):
        k = kinds[rng.integers(len(kinds))]
        a, b, c = (int(live[rng.integers(len(live))]) for _ in range(3))
        if k == _abi.CONST:
            a = int(rng.integers(2))
        ops.append((int(k), a, b, c, nxt))
        live.append(nxt)
        nxt += 1
    return ops


def _eval_plain(ops, vals):
    from paper_2407_19871_b200 import _abi
    v = dict(vals)
    f = {_abi.AND: lambda a, b: a & b, _abi.OR: lambda a, b: a | b, _abi.XOR: lambda a, b: a ^ b,
         _abi.XNOR: lambda a, b: 1 - (a ^ b), _abi.NAND: lambda a, b: 1 - (a & b),
         _abi.NOR: lambda a, b: 1 - (a | b), _abi.ANDNY: lambda a, b: (1 - a) & b,
         _abi.ORNY: lambda a, b: (1 - a) | b}
    for k, a, b, c, o in ops:
        if k in f:
            v[o] = f[k](v[a], v[b])
        elif k == _abi.MAJ:
            v[o] = 1 if v[a] + v[b] + v[c] >= 2 else 0
        elif k == _abi.XOR3:
            v[o] = v[a] ^ v[b] ^ v[c]
        elif k == _abi.MUX:
            v[o] = v[b] if v[a] else v[c]
        elif k == _abi.NOT:
            v[o] = 1 - v[a]
        elif k == _abi.COPY:
            v[o] = v[a]
        else:
            v[o] = a
    return v


@pytest.mark.parametrize("seed,level,n_in,n_ops", [(1, 80, 48, 400), (2, 80, 48, 400),
                                                  (3, 80, 48, 400), (4, 128, 600, 4000)])
def test_random_gate_programs_level_scheduled(dev, seed, level, n_in, n_ops):
    """The circuit scheduler (csrc/program.hpp) on random DAGs of every gate kind (incl.
    the flagged ANDNY / ORNY / MAJ): decrypted outputs equal plaintext evaluation; the
    plan's bootstrap count equals the accounting (MUX = 2 units, free gates 0).  The wide
    128-bit case puts > #SM bootstraps in a level (throughput kernel)."""
    from paper_2407_19871_b200 import _abi, plan
    p, keys, ctx = dev[level]
    rng = np.random.default_rng(seed)
    ops = _random_program(rng, n_in, n_ops, n_in)
    bits = rng.integers(0, 2, n_in).astype(np.uint8)
    ctx.pool_reserve(n_in + n_ops)
    ctx.h2d(0, keys.encrypt_bits(bits, 900 + seed))
    ctx.counters_reset()
    ctx.run(ops)
    want = _eval_plain(ops, {i: int(bits[i]) for i in range(n_in)})
    got = keys.decrypt_bits(ctx.d2h(n_in, n_ops))
    assert [int(x) for x in got] == [want[n_in + i] for i in range(n_ops)]
    units = sum(2 if k == _abi.MUX else (0 if k in (_abi.NOT, _abi.COPY, _abi.CONST) else 1)
                for k, *_ in ops)
    assert ctx.counters()["bootstrap_units"] == units
    assert plan(ops)["blind_rotations"] == units


def test_loc_pir_c_abi_entry(dev):
    """locpir_b200_loc_pir (the batched circuits.hpp:276-324 entry point) directly."""
    from paper_2407_19871_b200 import workloads as W
    p, keys, ctx = dev[128]
    b = W.make_batch(3, 5, 16, 4, seed=77)
    b.x[1] = (b.boxes[2, 0] + b.boxes[2, 1]) // 2
    b.y[1] = (b.boxes[2, 2] + b.boxes[2, 3]) // 2
    lay = W.PoolLayout(b)
    ctx.pool_reserve(lay.total)
    W.load_batch(ctx, keys, b, lay, seed=78)
    ctx.loc_pir(b.Q, b.R, b.l, b.m, lay.x, lay.y, lay.bnd, lay.svc, lay.out, lay.scratch)
    assert np.array_equal(W.read_results(ctx, keys, b, lay), b.truth())


@pytest.mark.parametrize("level,Q,R,l,m", [(128, 4, 9, 16, 8), (80, 3, 5, 13, 4)])
def test_folded_loc_pir_encrypted(dev, level, Q, R, l, m):
    """Flagged plaintext-boundary mode run encrypted: same decrypted
    result as the reference circuit, fewer bootstraps."""
    from paper_2407_19871_b200 import workloads as W
    p, keys, ctx = dev[level]
    b = W.make_batch(Q, R, l, m, seed=11 + level)
    for q in range(min(Q, R)):
        b.x[q] = (b.boxes[q, 0] + b.boxes[q, 1]) // 2
        b.y[q] = (b.boxes[q, 2] + b.boxes[q, 3]) // 2
    lay = W.PoolLayout(b)
    ctx.pool_reserve(lay.total)
    W.load_batch(ctx, keys, b, lay, seed=12)
    ctx.counters_reset()
    prog = W.program(ctx, b, lay, folded=True)
    prog.launch()
    assert np.array_equal(W.read_results(ctx, keys, b, lay), b.truth())
    assert ctx.counters()["bootstrap_units"] < b.units() // 2
    prog.close()


@pytest.mark.parametrize("count,first", [(1000, 7), (255, 3), (256, 0), (4097, 1)])
def test_pool_transfer_round_trip(dev, count, first):
    """Host<->pool copies: >= 256 rows go as one 1-D copy + repack/pack kernels (K4),
    fewer as a pitched 2-D copy; both must round-trip the wire layout exactly and leave
    neighbouring slots untouched."""
    p, keys, ctx = dev[128]
    ctx.pool_reserve(first + count + 2)
    rng = np.random.default_rng(count)
    guard = rng.integers(0, 2 ** 32, (first + count + 2, p.n + 1), dtype=np.uint64).astype(np.uint32)
    ctx.h2d(0, guard)
    rows = rng.integers(0, 2 ** 32, (count, p.n + 1), dtype=np.uint64).astype(np.uint32)
    ctx.h2d(first, rows)
    back = ctx.d2h(0, first + count + 2)
    assert np.array_equal(back[first:first + count], rows)
    assert np.array_equal(back[:first], guard[:first])
    assert np.array_equal(back[first + count:], guard[first + count:])


def test_empty_and_boundary_inputs(dev):
    """Zero-count calls are no-ops, out-of-range slots and bad arguments fail loudly."""
    from paper_2407_19871_b200 import _abi
    from paper_2407_19871_b200.engine import InvalidArgument
    p, keys, ctx = dev[128]
    ctx.pool_reserve(64)
    ctx.run([])                                               # empty program
    ctx.load_queries([], 16, [], [])                          # no payloads
    ctx.client_encrypt(keys.lwe_key, 1, np.zeros(0, np.uint32), first_slot=0)
    assert ctx.store_responses([], 4) == []
    with pytest.raises(InvalidArgument):                      # slot range past the pool
        ctx.h2d(ctx.pool_capacity, keys.encrypt_bits(np.ones(1, np.uint8), 1))
    with pytest.raises(InvalidArgument):
        ctx.client_encrypt(np.full(p.n, 2, np.uint8), 1, np.zeros(1, np.uint32), 0)
    with pytest.raises(InvalidArgument):
        ctx.store_responses([ctx.pool_capacity - 1], 4)
    with pytest.raises(InvalidArgument):                      # NOT of a never-written slot is fine,
        ctx.run([(_abi.AND, 0, 1, _abi.SLOT_NONE, 0)])       # but writing a slot it reads is not
    out = ctx.gate_batch_host(_abi.NAND, np.zeros((0, p.n + 1), np.uint32),
                              np.zeros((0, p.n + 1), np.uint32))
    assert out.shape == (0, p.n + 1)


@pytest.mark.parametrize("level", [80, 128])
def test_fft_rounding_margin(dev, level):
    """the pre-KS coefficients are exact iff every inverse-transform output
    lies within 1/2 of an integer; measure the worst distance over a full cfg2-sized batch
    at both parameter sets -- 65,536 blind rotations of uniform random inputs and 65,536
    of real NAND inputs -- and pin it far below 1/2.  (Adversarial maximum-magnitude
    digit inputs: tests/test_oracle_tfhe.py, on the oracle's identical arithmetic.)"""
    p, keys, ctx = dev[level]
    rng = np.random.default_rng(level + 1)
    G = 65536
    lwe = rng.integers(0, 2 ** 32, (G, p.n + 1), dtype=np.uint64).astype(np.uint32)
    bits = rng.integers(0, 2, (2, G)).astype(np.uint8)
    a, b = keys.encrypt_bits(bits[0], 3), keys.encrypt_bits(bits[1], 4)
    gate = (0 - a.astype(np.int64) - b.astype(np.int64)) & 0xFFFFFFFF
    gate[:, -1] = (gate[:, -1] + 0x20000000) & 0xFFFFFFFF  # NAND: (+1/8) - a - b
    e1 = ctx.debug_fft_error(lwe)
    e2 = ctx.debug_fft_error(gate.astype(np.uint32))
    print(f"FFT rounding margin ({level}-bit, {G} + {G} blind rotations): uniform {e1:.3e}, "
          f"NAND inputs {e2:.3e}")
    # 128-bit (Bgbit 7): a wide margin; 80-bit (Bgbit 10, digits to +-512): narrower but < 1/2
    assert 0.0 < max(e1, e2) < (0.25 if level == 80 else 1.0 / 16)


def test_program_graph_replay_survives_pool_growth(dev):
    """program_launch replays a CUDA graph after the first launch; growing the pool moves
    the device buffers, which must trigger a re-capture (stale pointers would corrupt)."""
    from paper_2407_19871_b200 import _abi
    p, keys, ctx = dev[128]
    G = 300
    ctx.pool_reserve(3 * G)
    rng = np.random.default_rng(11)
    A, B = rng.integers(0, 2, G).astype(np.uint8), rng.integers(0, 2, G).astype(np.uint8)
    ctx.h2d(0, keys.encrypt_bits(A, 5))
    ctx.h2d(G, keys.encrypt_bits(B, 6))
    prog = ctx.program([(_abi.XOR, g, G + g, _abi.SLOT_NONE, 2 * G + g) for g in range(G)])
    for rounds in range(3):                      # direct launch, then graph replays
        prog.launch()
        assert np.array_equal(keys.decrypt_bits(ctx.d2h(2 * G, G)), A ^ B)
    ctx.pool_reserve(ctx.pool_capacity * 4)      # reallocates (and copies) the pool
    ctx.h2d(2 * G, np.zeros((G, p.n + 1), np.uint32))
    prog.launch()
    assert np.array_equal(keys.decrypt_bits(ctx.d2h(2 * G, G)), A ^ B)
    prog.close()


@pytest.mark.parametrize("level", [80, 128])
def test_flagged_gate_forms_on_the_throughput_kernel(dev, level, okeys80, okeys128):
    """MAJ and XOR3 (3-input prologue), ANDNY and ORNY with more bootstraps per level than
    SMs, so the throughput kernel (not the latency kernel) runs them: bit-exact with the
    oracle."""
    from paper_2407_19871_b200 import _abi
    p, keys, ctx = dev[level]
    ok = okeys80 if level == 80 else okeys128
    G = 600
    rng = np.random.default_rng(level + 7)
    bits = rng.integers(0, 2, (3, G)).astype(np.uint8)
    cts = [keys.encrypt_bits(bits[i], 70 + i) for i in range(3)]
    ctx.pool_reserve(7 * G)
    for i in range(3):
        ctx.h2d(i * G, cts[i])
    ops = [(_abi.MAJ, g, G + g, 2 * G + g, 3 * G + g) for g in range(G)]
    ops += [(_abi.ANDNY, g, G + g, _abi.SLOT_NONE, 4 * G + g) for g in range(G)]
    ops += [(_abi.ORNY, g, G + g, _abi.SLOT_NONE, 5 * G + g) for g in range(G)]
    ops += [(_abi.XOR3, g, G + g, 2 * G + g, 6 * G + g) for g in range(G)]
    ctx.run(ops)
    a, b, c = bits
    for base, want, kind in ((3, (a.astype(int) + b + c >= 2), "maj"), (4, (1 - a) & b, "andny"),
                             (5, (1 - a) | b, "orny"), (6, a ^ b ^ c, "xor3")):
        got = ctx.d2h(base * G, G)
        assert list(keys.decrypt_bits(got)) == list(np.asarray(want, np.uint8)), kind
        for g in (0, G - 1):
            args = (cts[0][g], cts[1][g], cts[2][g]) if kind in ("maj", "xor3") else (cts[0][g], cts[1][g])
            assert np.array_equal(got[g], ok.gate(kind, *args)), kind


def test_python_mirror_majority_gate(dev):
    """GateEngine.hom_maj (flagged 3-input majority) through the Python mirror."""
    from paper_2407_19871_b200 import GateEngine
    p, keys, ctx = dev[80]
    eng = GateEngine(ctx, keys, seed=8)
    eng._next_slot = 0
    for a in (0, 1):
        for b in (0, 1):
            for c in (0, 1):
                ca, cb, cc = eng.encrypt(bool(a)), eng.encrypt(bool(b)), eng.encrypt(bool(c))
                assert eng.decrypt(eng.hom_maj(ca, cb, cc)) == (a + b + c >= 2)


def test_eager_and_level_batched_evaluation_give_identical_ciphertexts(dev):
    """acceptance.cpp:416-447 (worker invariance), restated for the level scheduler: the
    same loc_pir on the same input ciphertexts, evaluated gate by gate (one bootstrap per
    launch) and level-batched, yields bit-identical output ciphertexts."""
    from paper_2407_19871_b200 import GateEngine
    from paper_2407_19871_b200.circuits import (EncodedRegion, FixedPointFormat, PlainWord,
                                                ServiceCiphertext, constant_word, loc_pir)
    p, keys, ctx = dev[80]
    fmt = FixedPointFormat(4, 2)
    l = fmt.total_bits()
    rng = np.random.default_rng(31)
    qbits = rng.integers(0, 2, 2 * l).astype(np.uint8)
    sbits = rng.integers(0, 2, 2 * 3).astype(np.uint8)
    q_cts = keys.encrypt_bits(qbits, 41)
    s_cts = keys.encrypt_bits(sbits, 42)
    outs = []
    for batched in (False, True):
        eng = GateEngine(ctx, keys, seed=5)
        eng._next_slot = 0
        qb = eng.load(q_cts)
        sb = eng.load(s_cts)
        from paper_2407_19871_b200.circuits import CipherWord
        x, y = CipherWord(qb[:l], fmt), CipherWord(qb[l:], fmt)
        regions = []
        for i, (x1, x2, y1, y2) in enumerate(((-8, 6, -8, 8), (-3, 9, -10, 2))):
            w = [constant_word(PlainWord.from_integer(v, fmt), eng) for v in (x1, x2, y1, y2)]
            regions.append(EncodedRegion(*w, ServiceCiphertext(sb[3 * i:3 * i + 3]), i))
        if not batched:  # every gate runs as its own one-bootstrap launch
            import contextlib
            eng.batch = lambda: contextlib.nullcontext(eng)
        out = loc_pir(x, y, regions, eng, tree=True)
        outs.append(eng.samples(out.bits))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("name,R,kw", [("cfg3", 256, {}), ("cfg3", 256, {"folded": True}),
                                       ("cfg4", 16, {}), ("cfg5", 64, {}),
                                       ("cfg5", 64, {"maj": True})])
def test_loc_pir_program_every_ciphertext_equals_oracle(dev, okeys128, name, R, kw):
    """A whole LocPIR gate program on the B200 against the same program on the CPU oracle
    -- cfg3 at its stated size (1 query x 256 boxes, 66,304 bootstraps), one query of cfg4
    (16 boxes) and of cfg5 (64 boxes, encrypted boundaries, l = 32), reference circuit and
    flagged modes (oracle.run_program): EVERY ciphertext of the pool -- inputs, each comparator, mask and
    XOR-tree intermediate (a loc_pir program gives each its own slot) and the outputs -- is
    bit-exact, and the outputs decrypt to the plaintext answer."""
    import os
    from oracle import oracle as O
    from paper_2407_19871_b200 import workloads as W
    sec, _, _, l, m, enc = W.CONFIGS[name]
    p, keys, ctx = dev[128]
    b = W.make_batch(1, R, l, m, seed=300 + R, encrypted_bounds=enc)
    b.x[0] = (b.boxes[0, 0] + b.boxes[0, 1]) // 2
    b.y[0] = (b.boxes[0, 2] + b.boxes[0, 3]) // 2
    lay = W.PoolLayout(b)
    ctx.pool_reserve(lay.total)
    W.load_batch(ctx, keys, b, lay, seed=17)
    before = ctx.d2h(0, lay.total)
    ops = W.program_ops(b, lay, **kw)
    prog = ctx.program(ops)
    prog.launch()
    gpu = ctx.d2h(0, lay.total)
    prog.close()
    assert np.array_equal(W.read_results(ctx, keys, b, lay), b.truth())
    cpu = O.run_program(okeys128, ops, before.copy(), threads=os.cpu_count() or 1, simd="auto")
    written = sorted({o.out for o in ops})
    bad = [s for s in written if not np.array_equal(gpu[s], cpu[s])]
    assert not bad, f"{len(bad)} of {len(written)} program ciphertexts differ, first slots {bad[:5]}"


@pytest.mark.parametrize("count", [256, 4097])
def test_gate_batch_host_zero_copy_equals_copy_path(dev, okeys128, count):
    """gate_batch_host on pinned host buffers reads the inputs over PCIe inside the blind
    rotation (zero-copy); on pageable buffers it copies them first.  Both give the same
    ciphertexts, equal to the oracle's."""
    import torch
    from paper_2407_19871_b200 import _abi
    p, keys, ctx = dev[128]
    rng = np.random.default_rng(count)
    A = rng.integers(0, 2, count).astype(np.uint8)
    B = rng.integers(0, 2, count).astype(np.uint8)
    a = keys.encrypt_bits(A, 5)
    b = keys.encrypt_bits(B, 6)
    for kind, fn, name in ((_abi.NAND, lambda x, y: 1 - (x & y), "nand"),
                           (_abi.XOR, lambda x, y: x ^ y, "xor")):
        copied = ctx.gate_batch_host(kind, a, b)  # numpy: pageable -> copy path
        a_h = torch.from_numpy(a.view(np.int32)).pin_memory()
        b_h = torch.from_numpy(b.view(np.int32)).pin_memory()
        o_h = torch.empty(a_h.shape, dtype=torch.int32).pin_memory()
        ctx.gate_batch_host_ptr(kind, a_h.data_ptr(), b_h.data_ptr(), o_h.data_ptr(), count)
        zc = o_h.numpy().view(np.uint32)
        assert np.array_equal(zc, copied), name
        assert np.array_equal(keys.decrypt_bits(zc), fn(A, B)), name
        for g in (0, count - 1):
            assert np.array_equal(zc[g], okeys128.gate(name, a[g], b[g])), name
