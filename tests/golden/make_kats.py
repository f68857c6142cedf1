"""Per-stage known-answer vectors for the bootstrap path (SURVEY §8(c) "the builder must
generate KATs"): seeded keys, then the EXACT mod-2^32 oracle's outputs stage by stage
for a handful of gates at both parameter sets, written to tests/golden/stage_kats.npz.

  combined LWE (gate linear form, gate_engine.hpp:196-240 + NAND/ANDNY)
  -> abar (mod switch to [0, 2N))
  -> ACC after 1, 2 and 16 CMux steps (exact schoolbook external product)
  -> extracted N-dim LWE after all n steps (FP64-FFT mode, asserted == exact on the
     first 16 steps here and on whole rotations in tests/test_oracle_tfhe.py)
  -> key-switched n-dim LWE (= the gate output) -> decrypted bit.

Test infrastructure only.  Regenerate with:  python tests/golden/make_kats.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

KEY_SEED = 20240719
STEPS = (1, 2, 16)
# (name, off, c0, c1, bit_a, bit_b, expected bit)
CASES = [
    ("nand_1_1", 0x20000000, -1, -1, 1, 1, 0),
    ("and_1_0", 0xE0000000, 1, 1, 1, 0, 0),
    ("xor_0_1", 0x40000000, 2, 2, 0, 1, 1),
    ("andny_0_1", 0xE0000000, -1, 1, 0, 1, 1),
]


def combine(off, c0, c1, a, b):
    c = (np.int64(c0) * a.astype(np.int64) + np.int64(c1) * b.astype(np.int64)) & 0xFFFFFFFF
    c = c.astype(np.uint32)
    c[-1] = np.uint32((int(c[-1]) + off) & 0xFFFFFFFF)
    return c


def main():
    out = {}
    for level in (80, 128):
        K = O.TfheKeys(level, KEY_SEED)
        s = O.NoiseSampler(KEY_SEED + level, K.p.alpha_in)
        for name, off, c0, c1, ba, bb, want in CASES:
            a, b = K.encrypt(ba, s), K.encrypt(bb, s)
            comb = combine(off, c0, c1, a, b)
            pre = f"s{level}_{name}_"
            out[pre + "a"], out[pre + "b"], out[pre + "combined"] = a, b, comb
            out[pre + "abar"] = np.array([O.mod_switch(int(x), K.N) for x in comb], np.uint16)
            for k in STEPS:
                ex = K.blind_rotate_acc(comb, mode=O.EXACT, steps=k)
                assert np.array_equal(ex, K.blind_rotate_acc(comb, mode=O.FFT, steps=k))
                out[pre + f"acc{k}"] = ex
            ext = K.blind_rotate_extract(comb, mode=O.FFT)
            ks = K.keyswitch(ext)
            assert K.decrypt(ks) == want, (level, name)
            out[pre + "extracted"], out[pre + "ks"] = ext, ks
            out[pre + "meta"] = np.array([level, off, c0 & 0xFFFFFFFF, c1 & 0xFFFFFFFF, want],
                                         np.uint32)
    out["key_seed"] = np.array([KEY_SEED], np.uint64)
    path = os.path.join(HERE, "stage_kats.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(CASES) * 2, "cases")


if __name__ == "__main__":
    main()
