"""cfg1 (80-bit, 1 query x 1 box) and cfg3 (1 query x 256 boxes) program latency with
per-kernel-class times (kernel_stats), for latency-kernel A/B runs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2407_19871_b200 import ClientKeys, Context, TfheParams  # noqa: E402
from paper_2407_19871_b200 import workloads as W  # noqa: E402

for name in ("cfg1", "cfg1f", "cfg1t"):
    p = TfheParams(80)
    keys = ClientKeys(p, 20240719)
    ctx = Context(p, 0)
    ctx.upload_keys(keys.bk, keys.ksk)
    b = W.make_batch(1, 1, 16, 8, seed=3)
    b.x[0] = (b.boxes[0, 0] + b.boxes[0, 1]) // 2
    b.y[0] = (b.boxes[0, 2] + b.boxes[0, 3]) // 2
    lay = W.PoolLayout(b)
    ctx.pool_reserve(lay.total)
    W.load_batch(ctx, keys, b, lay, seed=4)
    prog = W.program(ctx, b, lay, folded=name != "cfg1", tree=name.endswith("t"))
    prog.launch()
    ctx.sync()
    reps = 20
    t = time.perf_counter()
    for _ in range(reps):
        prog.launch()
    ctx.sync()
    dt = (time.perf_counter() - t) / reps
    ok = np.array_equal(W.read_results(ctx, keys, b, lay), b.truth())
    print(f"{name}: {dt*1e3:.2f} ms/query  {1/dt:.1f} q/s  levels={prog.kernels}  correct={ok}")
    prog.close()
    ctx.close()
