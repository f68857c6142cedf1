"""Blind-rotation launch time per level size: the throughput kernel K1 (LOCPIR_B200_SMALL=0)
against the latency kernel K1l (default for levels <= #SMs), through debug_blind_rotate
with launch timing.  Prints one line per parameter set: count:ms pairs."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_19871_b200 import ClientKeys, Context, TfheParams  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "default"
counts = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else
                           "16,74,148,149,222,296,370,444,592").split(",")]
for level in (80, 128):
    p = TfheParams(level)
    keys = ClientKeys(p, 7)
    ctx = Context(p, 0)
    ctx.upload_keys(keys.bk, keys.ksk)
    rng = np.random.default_rng(1)
    row = []
    for count in counts:
        lwe = rng.integers(0, 2 ** 32, (count, p.n + 1), dtype=np.uint64).astype(np.uint32)
        ctx.debug_blind_rotate(lwe)
        ctx.timing(True)
        for _ in range(3):
            ctx.debug_blind_rotate(lwe)
        ms, n = ctx.kernel_stats()["blind_rotate"]
        ctx.timing(False)
        row.append(f"{count}:{ms / max(n, 1):.2f}")
    print(tag, level, " ".join(row), flush=True)
    ctx.close()
