"""Host-side checks of the product library: it loads, exports every symbol the C
ABI header declares, and its host-only pieces (client key material, encryption,
circuit scheduler) agree with the oracle and the reference -- no GPU needed."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "locpir_b200.h")).read()
    return sorted(set(re.findall(r"\b(locpir_b200_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    from paper_2407_19871_b200 import _abi
    so = _abi.LIB_PATH
    assert os.path.exists(so)
    nm = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True,
                        check=True).stdout
    exported = set(re.findall(r"\bT (locpir_b200_\w+)", nm))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing
    bound = {name for name, _, _ in _abi.SIGNATURES}
    assert set(header_symbols()) <= bound


def test_cuda_code_is_sm100a():
    from paper_2407_19871_b200 import _abi
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_engine_kind_parsing():
    from paper_2407_19871_b200 import InvalidArgument, parse_engine_kind
    assert parse_engine_kind("clear") == "clear"
    assert parse_engine_kind("tlwe-oracle") == "tlwe-oracle"
    assert parse_engine_kind("tfhe-b200") == "tfhe-b200"
    with pytest.raises(InvalidArgument):  # test_gate_engine.cpp:154
        parse_engine_kind("tfhe")


@pytest.mark.parametrize("level", [80, 128])
def test_product_keygen_equals_oracle(level, okeys80, okeys128):
    from paper_2407_19871_b200 import ClientKeys, TfheParams
    ok = okeys80 if level == 80 else okeys128
    k = ClientKeys(TfheParams(level), 7)
    assert np.array_equal(k.lwe_key, ok.lwe_key)
    assert np.array_equal(k.trlwe_key, ok.trlwe_key)
    assert np.array_equal(k.bk, ok.bk())
    assert np.array_equal(k.ksk, ok.ksk())


def test_product_encrypt_decrypt_equal_oracle(oracle, okeys128):
    from paper_2407_19871_b200 import ClientKeys, TfheParams
    k = ClientKeys(TfheParams(128), 7, evaluation_keys=False)
    bits = [1, 0, 0, 1, 1]
    cts = k.encrypt_bits(bits, 99)
    s = oracle.NoiseSampler(99, okeys128.p.alpha_in)
    ref = np.stack([okeys128.encrypt(b, s) for b in bits])
    assert np.array_equal(cts, ref)
    assert list(k.decrypt_bits(cts)) == bits


def test_param_sets():
    from paper_2407_19871_b200 import TfheParams
    p = TfheParams(128)
    assert (p.c.n, p.c.N, p.c.k, p.c.bk_l, p.c.bk_bgbit, p.c.ks_t, p.c.ks_basebit) == \
        (630, 1024, 1, 3, 7, 8, 2)
    assert p.c.alpha_in == 2 ** -15 and p.c.alpha_bk == 2 ** -25
    assert p.sample_bytes() == 2524  # acceptance.cpp:59
    q = TfheParams(80)
    assert (q.c.n, q.c.bk_l, q.c.bk_bgbit) == (500, 2, 10)
    assert p.bk_words() * 8 == 61931520  # SURVEY §8(a') |BK_freq|
    assert p.ksk_words() * 4 == 62029824


def _slots(Q, R, l, m):
    x = np.arange(Q * l).reshape(Q, l)
    y = Q * l + np.arange(Q * l).reshape(Q, l)
    b = 2 * Q * l + np.arange(R * 4 * l).reshape(R, 4, l)
    s = 2 * Q * l + R * 4 * l + np.arange(R * m).reshape(R, m)
    o = s.max() + 1 + np.arange(Q * m).reshape(Q, m)
    return x, y, b, s, o, int(o.max() + 1)


@pytest.mark.parametrize("tree", [False, True])
@pytest.mark.parametrize("N,l,m", [(1, 16, 8), (3, 6, 3), (9, 16, 9), (16, 16, 8), (256, 16, 32)])
def test_loc_pir_program_gate_counts(N, l, m, tree):
    """N(12l + 2m + 3) units (bench.hpp:35-43) and N(8l + 2m + 3) key switches."""
    from paper_2407_19871_b200 import loc_pir_program, plan
    from paper_2407_19871_b200.circuits import predict_gate_units
    x, y, b, s, o, first = _slots(1, N, l, m)
    ops = loc_pir_program(1, N, l, m, x, y, b, s, o, first, tree)
    pl = plan([(op.kind, op.in0, op.in1, op.in2, op.out) for op in ops])
    assert pl["blind_rotations"] == predict_gate_units(N, l, m)
    assert pl["key_switches"] == N * (8 * l + 2 * m + 3)
    depth = (l + 1) + 3 + (int(np.ceil(np.log2(N))) + 1 if tree else N)
    assert pl["levels"] == depth


def test_loc_pir_counts_match_reference_golden(golden):
    from paper_2407_19871_b200 import loc_pir_program, plan
    rows = np.array(golden["locpir_synthetic_N_l_m_got_expected_units_xnor_mux_and_xor_not_pred"])
    rows = rows.reshape(-1, 12)
    for N, l, m, got, exp, units, xnor, mux, and_, xor, nots, pred in rows:
        assert got == exp and units == pred
        x, y, b, s, o, first = _slots(1, N, l, m)
        ops = loc_pir_program(1, int(N), int(l), int(m), x, y, b, s, o, first, False)
        kinds = np.array([op.kind for op in ops])
        assert (kinds == 3).sum() == xnor and (kinds == 5).sum() == mux
        assert (kinds == 0).sum() == and_ and (kinds == 2).sum() == xor
        assert (kinds == 6).sum() == nots
        assert plan([(op.kind, op.in0, op.in1, op.in2, op.out) for op in ops])[
            "blind_rotations"] == units


def test_scheduler_rejects_malformed_programs():
    from paper_2407_19871_b200 import InvalidArgument, plan
    with pytest.raises(InvalidArgument):
        plan([(0, 0, 1, 0, 5), (0, 2, 3, 0, 5)])   # slot written twice
    with pytest.raises(InvalidArgument):
        plan([(0, 0, 1, 0, 5), (0, 2, 3, 0, 1)])   # write after read
    with pytest.raises(InvalidArgument):
        plan([(42, 0, 1, 0, 5)])                   # unknown kind


def test_scheduler_levels_and_mux_split():
    from paper_2407_19871_b200 import plan
    # comparator-like chain: t1_i independent, t0 chain through MUX "then" half only
    ops, t0 = [], 100
    ops.append((9, 0, 0, 0, t0))  # CONST 0
    for i in range(4):
        ops.append((3, i, 10 + i, 0, 200 + i))              # XNOR
        ops.append((5, 200 + i, t0, 10 + i, 300 + i))       # MUX
        t0 = 300 + i
    pl = plan(ops)
    assert pl["levels"] == 5 and pl["blind_rotations"] == 12 and pl["key_switches"] == 8


def test_plan_wave_structure_random_programs():
    """Host-only: for random SSA programs the scheduler's level count equals the longest
    bootstrap path (free gates do not add levels unless chained) and never exceeds the
    op count; malformed inputs raise."""
    import numpy as np
    from paper_2407_19871_b200 import plan
    rng = np.random.default_rng(5)
    for trial in range(20):
        n_in, n_ops = 16, 60
        ops, depth, nxt = [], {i: 0 for i in range(n_in)}, n_in
        for _ in range(n_ops):
            k = int(rng.choice([0, 1, 2, 3, 4]))  # bootstrapped two-input gates
            a, b = int(rng.integers(nxt)), int(rng.integers(nxt))
            ops.append((k, a, b, 0, nxt))
            depth[nxt] = max(depth[a], depth[b]) + 1
            nxt += 1
        pl = plan(ops)
        assert pl["levels"] == max(depth.values())
        assert pl["blind_rotations"] == n_ops == pl["key_switches"]


def test_ctx_rejects_parameters_the_kernels_are_not_built_for():
    """ctx_create checks the parameter set before touching the GPU: n beyond the key
    switch's 640-column coverage and gadget shapes without a kernel instantiation."""
    import ctypes as C
    from paper_2407_19871_b200 import _abi
    L = _abi.lib()
    for n, l, bg in ((700, 3, 7), (630, 4, 6)):
        p = _abi.Params()
        assert L.locpir_b200_params_default(128, C.byref(p)) == 0
        p.n, p.bk_l, p.bk_bgbit = n, l, bg
        h = C.c_void_p()
        assert L.locpir_b200_ctx_create(C.byref(p), 0, None, C.byref(h)) == _abi.EINVAL
        assert not h.value


def test_key_blob_roundtrip(tmp_path):
    """BK/KSK blobs persisted in torus form (skip keygen); secret-less server
    files; tampering and truncation are rejected."""
    from paper_2407_19871_b200 import ClientKeys, TfheParams
    from paper_2407_19871_b200.engine import InvalidArgument
    k = ClientKeys(TfheParams(80), 5)
    f = tmp_path / "k.bin"
    k.save(str(f))
    r = ClientKeys.load(str(f))
    assert r.params.security_bits == 80
    for a in ("lwe_key", "trlwe_key", "bk", "ksk"):
        assert np.array_equal(getattr(r, a), getattr(k, a))
    bits = np.array([1, 0, 1], np.uint8)
    assert list(r.decrypt_bits(k.encrypt_bits(bits, 3))) == list(bits)
    pub = tmp_path / "pub.bin"
    k.save(str(pub), secret=False)
    p = ClientKeys.load(str(pub))
    assert p.lwe_key is None and np.array_equal(p.bk, k.bk)
    raw = bytearray(f.read_bytes())
    raw[100] ^= 1
    f.write_bytes(bytes(raw))
    with pytest.raises(InvalidArgument, match="checksum"):
        ClientKeys.load(str(f))
    f.write_bytes(b"junk")
    with pytest.raises(InvalidArgument, match="not a locpir_b200 key file"):
        ClientKeys.load(str(f))
