"""One cfg4-shaped LocPIR batch (128-bit, 64 queries x 16 boxes, l=16, m=8) through the
level-scheduled program -- for the per-wave launch list (BR / KS / LIN per level)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2407_19871_b200 import ClientKeys, Context, TfheParams  # noqa: E402
from paper_2407_19871_b200 import workloads as W  # noqa: E402

p = TfheParams(128)
keys = ClientKeys(p, 20240719)
ctx = Context(p, 0)
ctx.upload_keys(keys.bk, keys.ksk)
b = W.make_batch(64, 16, 16, 8, seed=5)
for q in range(16):
    b.x[q] = (b.boxes[q, 0] + b.boxes[q, 1]) // 2
    b.y[q] = (b.boxes[q, 2] + b.boxes[q, 3]) // 2
lay = W.PoolLayout(b)
ctx.pool_reserve(lay.total)
W.load_batch(ctx, keys, b, lay, seed=6)
prog = W.program(ctx, b, lay)
prog.launch()
ctx.sync()
ok = np.array_equal(W.read_results(ctx, keys, b, lay), b.truth())
print("cfg4-shaped batch correct:", ok, "launches:", prog.kernels)
sys.exit(0 if ok else 1)
