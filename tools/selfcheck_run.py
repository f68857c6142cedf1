"""Deterministic workload over every product kernel (tools/sanitize_run.py's coverage:
K0, K1 / K1l, K2t / K2 / K2s, K3, K4, K5 and client encryption) at one parameter set; prints
one line "digest <sha256>" over ALL outputs.  tools/selfcheck.sh runs it with the default
and the checked library (LPB_CHECKS device asserts + LPB_JITTER barrier jitter), several
LOCPIR_B200_POISON patterns for fresh pool / scratch / shared memory, and both kernel
choices (LOCPIR_B200_SMALL): every digest must be identical.  A bounds violation aborts
(device assert); a read of memory the kernel did not write, or a missing barrier, shows
up as a digest that changes with the poison or the jitter.  This stands in for
compute-sanitizer, which is closed on the GPU pool."""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    from paper_2407_19871_b200 import ClientKeys, Context, TfheParams, _abi
    from paper_2407_19871_b200 import workloads as W
    from paper_2407_19871_b200.server import BatchingServer
    from oracle import oracle as O
    from test_wire import query_payload, zero_sheet_payload
    level = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    G = 300
    h = hashlib.sha256()
    p = TfheParams(level)
    keys = ClientKeys(p, 9)
    ctx = Context(p, 0)
    ctx.upload_keys(keys.bk, keys.ksk)
    rng = np.random.default_rng(1)
    A = rng.integers(0, 2, G).astype(np.uint8)
    B = rng.integers(0, 2, G).astype(np.uint8)
    a, b = keys.encrypt_bits(A, 2), keys.encrypt_bits(B, 3)
    for kind, fn in ((_abi.NAND, lambda x, y: 1 - (x & y)), (_abi.XOR, lambda x, y: x ^ y)):
        out = ctx.gate_batch_host(kind, a, b)
        assert np.array_equal(keys.decrypt_bits(out), fn(A, B))
        h.update(out.tobytes())
    # a level that runs K1 (not K1l) and the tensor-core key switch K2t in both kernel
    # choices
    G2 = 1280
    A2 = rng.integers(0, 2, G2).astype(np.uint8)
    B2 = rng.integers(0, 2, G2).astype(np.uint8)
    a2, b2 = keys.encrypt_bits(A2, 4), keys.encrypt_bits(B2, 5)
    out = ctx.gate_batch_host(_abi.NAND, a2, b2)
    assert np.array_equal(keys.decrypt_bits(out), 1 - (A2 & B2))
    h.update(out.tobytes())
    # the zero-copy path (pinned inputs read over PCIe by the blind rotation's prologue)
    import torch
    ah = torch.from_numpy(a2.view(np.int32)).pin_memory()
    bh = torch.from_numpy(b2.view(np.int32)).pin_memory()
    oh = torch.empty(ah.shape, dtype=torch.int32).pin_memory()
    ctx.gate_batch_host_ptr(_abi.NAND, ah.data_ptr(), bh.data_ptr(), oh.data_ptr(), G2)
    assert np.array_equal(oh.numpy().view(np.uint32), out)
    # a small loc_pir batch (comparator chains, masks, XOR tree; K1l/K2s levels and K3)
    bt = W.make_batch(3, 4, 8, 3, seed=5)
    bt.x[0] = (bt.boxes[0, 0] + bt.boxes[0, 1]) // 2
    bt.y[0] = (bt.boxes[0, 2] + bt.boxes[0, 3]) // 2
    lay = W.PoolLayout(bt)
    ctx.pool_reserve(lay.total)
    W.load_batch(ctx, keys, bt, lay, 7)
    prog = W.program(ctx, bt, lay)
    prog.launch()
    prog.launch()  # graph replay
    assert np.array_equal(W.read_results(ctx, keys, bt, lay), bt.truth())
    h.update(ctx.d2h(int(lay.out.min()), bt.Q * bt.m).tobytes())
    prog.close()
    # the flagged folded mode (ANDNY / ORNY chains, ternary XOR3 sums) and a level of the
    # 3-input gates MAJ / XOR3 (the 3-input prologue)
    prog = W.program(ctx, bt, lay, folded=True)
    prog.launch()
    assert np.array_equal(W.read_results(ctx, keys, bt, lay), bt.truth())
    h.update(ctx.d2h(int(lay.out.min()), bt.Q * bt.m).tobytes())
    prog.close()
    G3 = 200
    base = lay.total - 4 * G3
    C3 = rng.integers(0, 2, (3, G3)).astype(np.uint8)
    for i in range(3):
        ctx.h2d(base + i * G3, keys.encrypt_bits(C3[i], 60 + i))
    ctx.run([(_abi.MAJ if g % 2 else _abi.XOR3, base + g, base + G3 + g, base + 2 * G3 + g,
              base + 3 * G3 + g) for g in range(G3)])
    out3 = ctx.d2h(base + 3 * G3, G3)
    want3 = np.where(np.arange(G3) % 2 == 1, (C3.sum(0) >= 2).astype(np.uint8), C3[0] ^ C3[1] ^ C3[2])
    assert np.array_equal(keys.decrypt_bits(out3), want3)
    h.update(out3.tobytes())
    # the batcher's wire kernels (K5)
    l, m = 8, 3
    boxes = np.array([[0, 20, 0, 20], [-10, 5, -10, 5]], np.int64)
    srv = BatchingServer(ctx, boxes, [5, 2], l, m, max_sessions=1, base_slot=lay.total)
    key = O.keygen_bits(p.n, 9)
    alpha = 2.0 ** -15 if level == 128 else 2.44e-5
    sheet, _ = zero_sheet_payload(key, O.NoiseSampler(30, alpha), 2, m)
    sid = srv.open_session(sheet)
    t = srv.submit(sid, query_payload(key, O.NoiseSampler(31, alpha), 3, 4, l)[0])
    srv.flush()
    resp = srv.take_response(t)
    rows = np.frombuffer(resp, "<u4").reshape(m, p.n + 1)
    assert sum(int(keys.decrypt_bits(rows[j])[0]) << j for j in range(m)) == 5 ^ 2
    h.update(resp)
    srv.close()
    # client-side encryption on the device
    mus = np.where(rng.integers(0, 2, 16) == 1, 0x20000000, 0xE0000000).astype(np.uint32)
    ctx.client_encrypt(keys.lwe_key, 77, mus, 0)
    enc = ctx.d2h(0, 16)
    assert list(keys.decrypt_bits(enc)) == list((mus == 0x20000000).astype(int))
    h.update(enc.tobytes())
    ctx.close()
    print(f"digest {level} {h.hexdigest()}")


if __name__ == "__main__":
    main()
