"""Stage-by-stage known answers (tests/golden/stage_kats.npz, made by make_kats.py from the
exact oracle): the oracle must reproduce every stage from the stored inputs with keys
regenerated from the seed; the B200 path must reproduce the extracted LWE, the key-switch
output and the gate output bit for bit (SURVEY §8(c) parity ladder)."""
import os

import numpy as np
import pytest

from oracle import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
KATS = np.load(os.path.join(HERE, "golden", "stage_kats.npz"))
SEED = int(KATS["key_seed"][0])
CASES = sorted({k[: k.rindex("_")] for k in KATS.files if k.endswith("_meta")})


@pytest.fixture(scope="module")
def okeys():
    return {lvl: O.TfheKeys(lvl, SEED) for lvl in (80, 128)}


def test_kat_file_covers_both_parameter_sets():
    assert len(CASES) == 8
    assert {int(KATS[c + "_meta"][0]) for c in CASES} == {80, 128}


@pytest.mark.parametrize("case", CASES)
def test_oracle_reproduces_every_stage(okeys, case):
    meta = KATS[case + "_meta"]
    K = okeys[int(meta[0])]
    comb = KATS[case + "_combined"]
    abar = np.array([O.mod_switch(int(x), K.N) for x in comb], np.uint16)
    assert np.array_equal(abar, KATS[case + "_abar"])
    for k in (1, 2, 16):
        assert np.array_equal(K.blind_rotate_acc(comb, mode=O.EXACT, steps=k), KATS[case + f"_acc{k}"])
    ext = K.blind_rotate_extract(comb, mode=O.FFT)
    assert np.array_equal(ext, KATS[case + "_extracted"])
    ks = K.keyswitch(ext)
    assert np.array_equal(ks, KATS[case + "_ks"])
    assert K.decrypt(ks) == int(meta[4])


@pytest.mark.gpu
@pytest.mark.parametrize("level", [80, 128])
def test_b200_reproduces_stage_kats(level):
    from paper_2407_19871_b200 import ClientKeys, Context, TfheParams
    p = TfheParams(level)
    keys = ClientKeys(p, SEED)
    ctx = Context(p, 0)
    ctx.upload_keys(keys.bk, keys.ksk)
    cases = [c for c in CASES if int(KATS[c + "_meta"][0]) == level]
    comb = np.stack([KATS[c + "_combined"] for c in cases])
    ext = ctx.debug_blind_rotate(comb)
    ks = ctx.debug_keyswitch(np.stack([KATS[c + "_extracted"] for c in cases]))
    for i, c in enumerate(cases):
        assert np.array_equal(ext[i], KATS[c + "_extracted"]), c
        assert np.array_equal(ks[i], KATS[c + "_ks"]), c
    # the whole gate through the pool and the scheduler
    from paper_2407_19871_b200 import _abi
    kinds = {"nand": _abi.NAND, "and": _abi.AND, "xor": _abi.XOR, "andny": _abi.ANDNY}
    ctx.pool_reserve(3 * len(cases))
    ctx.h2d(0, np.stack([KATS[c + "_a"] for c in cases]))
    ctx.h2d(len(cases), np.stack([KATS[c + "_b"] for c in cases]))
    ops = [(kinds[c.split("_")[1]], i, len(cases) + i, _abi.SLOT_NONE, 2 * len(cases) + i)
           for i, c in enumerate(cases)]
    ctx.run(ops)
    got = ctx.d2h(2 * len(cases), len(cases))
    for i, c in enumerate(cases):
        assert np.array_equal(got[i], KATS[c + "_ks"]), c
    ctx.close()
