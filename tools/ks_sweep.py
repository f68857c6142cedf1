"""Key-switch launch time per level size (128-bit and 80-bit): K2t vs the split path K2s,
through debug_keyswitch with launch timing.  Run once per library build (LOCPIR_B200_LIB)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_19871_b200 import ClientKeys, Context, TfheParams  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "base"
for level in (80, 128):
    p = TfheParams(level)
    keys = ClientKeys(p, 7)
    ctx = Context(p, 0)
    ctx.upload_keys(keys.bk, keys.ksk)
    rng = np.random.default_rng(1)
    row = []
    for count in (16, 48, 96, 128, 192, 256, 384, 512, 768, 1024, 1183):
        lweN = rng.integers(0, 2 ** 32, (count, p.N + 1), dtype=np.uint64).astype(np.uint32)
        ctx.debug_keyswitch(lweN)
        ctx.timing(True)
        for _ in range(5):
            ctx.debug_keyswitch(lweN)
        ms, n = ctx.kernel_stats()["keyswitch"]
        ctx.timing(False)
        row.append(f"{count}:{ms / max(n, 1):.3f}")
    print(tag, level, " ".join(row), flush=True)
    ctx.close()
