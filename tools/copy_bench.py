"""H2D/D2H rates: the pool's strided copy (cudaMemcpy2DAsync, 2,524 B rows into a 2,528 B
pitch) against a plain 1-D copy of the same bytes, pinned host memory, and the host-side
planning cost of a 65,536-gate batch."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2407_19871_b200 import Context, TfheParams, _abi
from paper_2407_19871_b200.engine import plan

p = TfheParams(128)
ctx = Context(p, 0, stream=torch.cuda.current_stream().cuda_stream)
n = 131072
ctx.pool_reserve(3 * 65536)
host = torch.empty((n, p.n + 1), dtype=torch.int32, pin_memory=True)
dev = torch.empty((n, p.n + 1), dtype=torch.int32, device="cuda")
ptr = C.c_void_p(host.data_ptr())
L = _abi.lib()
for name, fn in [("2d h2d", lambda: L.locpir_b200_pool_h2d(ctx.h, 0, n, ptr)),
                 ("1d h2d", lambda: dev.copy_(host, non_blocking=True)),
                 ("2d d2h", lambda: L.locpir_b200_pool_d2h(ctx.h, 0, n, ptr)),
                 ("1d d2h", lambda: host.copy_(dev, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"{name}: {dt*1e3:.2f} ms  {host.numel()*4/dt/1e9:.1f} GB/s")
ops = (_abi.GateOp * 65536)(*[_abi.GateOp(_abi.NAND, g, 65536 + g, _abi.SLOT_NONE, 131072 + g)
                              for g in range(65536)])
for _ in range(3):
    t = time.perf_counter(); plan(ops); print(f"plan 65,536 gates: {(time.perf_counter()-t)*1e3:.2f} ms")
