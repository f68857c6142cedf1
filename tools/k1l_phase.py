"""K1l phase breakdown (diagnostic build, LOCPIR_B200_LIB=lib_phclk.so): one small NAND
level at 80 and 128 bits; the kernel prints clock64 sums per CMux-step phase."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2407_19871_b200 import ClientKeys, Context, TfheParams, _abi  # noqa: E402

for sec in (80, 128):
    p = TfheParams(sec)
    keys = ClientKeys(p, 5)
    ctx = Context(p, 0)
    ctx.upload_keys(keys.bk, keys.ksk)
    G = int(os.environ.get("K1L_G", "64"))
    rng = np.random.default_rng(1)
    A = rng.integers(0, 2, G).astype(np.uint8)
    B = rng.integers(0, 2, G).astype(np.uint8)
    out = ctx.gate_batch_host(_abi.NAND, keys.encrypt_bits(A, 2), keys.encrypt_bits(B, 3))
    ctx.sync()
    print(sec, "correct", bool(np.array_equal(keys.decrypt_bits(out), 1 - (A & B))), flush=True)
    ctx.close()
