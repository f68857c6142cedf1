"""Pins the CPU oracle's LWE layer to vectors produced by the UNMODIFIED reference
(tests/golden/ref_vectors.json, made by tests/golden/make_golden.py from
oracle/_ref/ref_driver).  Anchors: torus.hpp:119-194, gate_engine.hpp:117-123."""
import numpy as np


def test_keygen_matches_reference(oracle, golden):
    assert list(oracle.keygen_bits(540, 11)) == golden["keygen_sec80_seed11"]
    assert list(oracle.keygen_bits(630, 12)) == golden["keygen_sec128_seed12"]
    assert list(oracle.keygen_bits(630, 7)) == golden["keygen_n630_seed7"]


def test_noise_sampler_streams_match_reference(oracle, golden):
    s = oracle.NoiseSampler(13, 2 ** -20.2)
    g, u = [], []
    for _ in range(64):
        g.append(s.gaussian())
        u.append(s.uniform())
    assert g == golden["sampler13_sec80_gauss"]
    assert u == golden["sampler13_sec80_unif"]
    s = oracle.NoiseSampler(99, 2 ** -15)
    assert [s.gaussian() for _ in range(256)] == golden["sampler99_a15_gauss"]
    s = oracle.NoiseSampler(5, 2 ** -25)
    assert [s.gaussian() for _ in range(256)] == golden["sampler5_a25_gauss"]


def test_encryption_matches_reference(oracle, golden):
    key = oracle.keygen_bits(630, 12)
    s = oracle.NoiseSampler(14, 2 ** -13.8)
    assert list(oracle.encrypt_bit(1, key, s)) == golden["enc_sec128_k12_s14_bit1"]
    assert list(oracle.encrypt_bit(0, key, s)) == golden["enc_sec128_k12_s14_bit0"]
    assert list(oracle.encrypt_torus(0, key, s)) == golden["enc_sec128_k12_s14_mu0"]
    a = oracle.encrypt_bit(1, key, s)
    assert oracle.phase(a, key) == golden["phase_of_next"][0]
    assert list(oracle.bootstrap_standin(a, key, s)) == golden["standin_refresh_of_next"]
    key = oracle.keygen_bits(630, 7)
    s = oracle.NoiseSampler(8, 2 ** -15)
    four = np.concatenate([oracle.encrypt_bit(i & 1, key, s) for i in range(4)])
    assert list(four) == golden["enc_n630_a15_k7_s8_four"]


def test_sample_sizes_match_reference(golden):
    # torus.hpp:227-230: 4(n+1) bytes; 2164 / 2524 (acceptance.cpp:58-59)
    assert golden["sample_bytes_sec80_sec128"] == [4 * 541, 4 * 631]


def test_standin_sign_rule(oracle):
    # gate_engine.hpp:117-123 / test_gate_engine.cpp:99-113 (oracle-engine-only KAT)
    key = oracle.keygen_bits(8, 2)
    s = oracle.NoiseSampler(3, 0.0)

    def th(raw):
        ct = np.zeros(9, np.uint32)
        ct[8] = raw
        return oracle.decrypt_bit(oracle.bootstrap_standin(ct, key, s), key)
    assert th(0x00000001) == 1
    assert th(0x80000000) == 1
    assert th(0x80000001) == 0
    assert th(0) == 0


def test_reference_truth_table_and_counters(golden):
    # the reference oracle engine's decrypted truth tables (gate_engine.hpp:196-269)
    t = golden["truth_table_and_or_xor_xnor_not_mux0_mux1"]
    i = 0
    for a in (0, 1):
        for b in (0, 1):
            assert t[i:i + 7] == [a & b, a | b, a ^ b, 1 - (a ^ b), 1 - a, b, a]
            i += 7
    assert golden["truth_table_counters"] == [4, 4, 4, 4, 4, 8, 32]
