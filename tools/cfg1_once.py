"""One BASELINE configs[0] LocPIR query (80-bit, 1 box) -- used for profiling the
small-level (latency) kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2407_19871_b200 import ClientKeys, Context, TfheParams  # noqa: E402
from paper_2407_19871_b200 import workloads as W  # noqa: E402

p = TfheParams(80)
keys = ClientKeys(p, 20240719)
ctx = Context(p, 0)
ctx.upload_keys(keys.bk, keys.ksk)
b = W.make_batch(1, 1, 16, 8, seed=3)
lay = W.PoolLayout(b)
ctx.pool_reserve(lay.total)
W.load_batch(ctx, keys, b, lay, seed=4)
prog = W.program(ctx, b, lay)
prog.launch()
ctx.sync()
ok = np.array_equal(W.read_results(ctx, keys, b, lay), b.truth())
print("cfg1 query correct:", ok)
sys.exit(0 if ok else 1)
