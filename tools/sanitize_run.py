"""Small workload that launches every product kernel once, for compute-sanitizer
(memcheck / racecheck / synccheck; one tool per gpurun call, tools/sanitize.sh):

  K0 k_bk_to_freq (key upload), K1 k_blind_rotate and K2 k_keyswitch (LOCPIR_B200_SMALL=0
  forces the throughput kernels on a small batch), K1l k_blind_rotate_lat and K2s
  k_keyswitch_split + k_ks_reduce (small levels), K3 k_linear (NOT / CONST), K4
  k_repack_rows / k_pack_rows (>= 256-row copies), K5 k_unpack_queries /
  k_load_zero_sheet / k_pack_responses (the batcher), k_client_encrypt.

Every result is checked, so a sanitizer run that perturbs nothing still proves the
kernels computed the right thing under instrumentation.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    from paper_2407_19871_b200 import ClientKeys, Context, TfheParams, _abi
    from paper_2407_19871_b200.server import BatchingServer
    level = int(os.environ.get("SAN_LEVEL", "80"))
    G = int(os.environ.get("SAN_GATES", "300"))
    p = TfheParams(level)
    keys = ClientKeys(p, 9)
    ctx = Context(p, 0)
    ctx.upload_keys(keys.bk, keys.ksk)                               # K0
    rng = np.random.default_rng(1)
    A = rng.integers(0, 2, G).astype(np.uint8)
    B = rng.integers(0, 2, G).astype(np.uint8)
    a, b = keys.encrypt_bits(A, 2), keys.encrypt_bits(B, 3)
    out = ctx.gate_batch_host(_abi.NAND, a, b)                       # K1/K1l + K2/K2s, K4
    assert np.array_equal(keys.decrypt_bits(out), 1 - (A & B)), "NAND"
    # free gates and a MUX (K3; both blind rotations of the MUX and one key switch)
    ctx.pool_reserve(8)
    ctx.h2d(0, keys.encrypt_bits(np.array([1, 0, 1], np.uint8), 4))
    ctx.run([(_abi.CONST, 1, _abi.SLOT_NONE, _abi.SLOT_NONE, 3),
             (_abi.NOT, 1, _abi.SLOT_NONE, _abi.SLOT_NONE, 4),
             (_abi.MUX, 0, 1, 3, 5)])
    assert list(keys.decrypt_bits(ctx.d2h(3, 3))) == [1, 1, 0], "CONST/NOT/MUX"
    # the batcher's wire kernels (K5) on one small session
    if os.environ.get("SAN_SERVER", "1") == "1":
        from oracle import oracle as O
        from test_wire import query_payload, zero_sheet_payload
        l, m = 8, 3
        boxes = np.array([[0, 20, 0, 20], [-10, 5, -10, 5]], np.int64)
        srv = BatchingServer(ctx, boxes, [5, 2], l, m, max_sessions=1, base_slot=1024)
        key = O.keygen_bits(p.n, 9)
        alpha = 2.0 ** -15 if level == 128 else 2.44e-5
        sheet, _ = zero_sheet_payload(key, O.NoiseSampler(30, alpha), 2, m)
        sid = srv.open_session(sheet)
        t = srv.submit(sid, query_payload(key, O.NoiseSampler(31, alpha), 3, 4, l)[0])
        srv.flush()
        rows = np.frombuffer(srv.take_response(t), "<u4").reshape(m, p.n + 1)
        got = sum(int(keys.decrypt_bits(rows[j])[0]) << j for j in range(m))
        assert got == 5 ^ 2, got
        srv.close()
    # client-side encryption on the device
    ctx.pool_reserve(64)
    mus = np.where(rng.integers(0, 2, 16) == 1, 0x20000000, 0xE0000000).astype(np.uint32)
    ctx.client_encrypt(keys.lwe_key, 77, mus, 32)
    assert list(keys.decrypt_bits(ctx.d2h(32, 16))) == list((mus == 0x20000000).astype(int))
    ctx.close()
    print(f"sanitize workload ok ({level}-bit, {G} gates, SMALL={os.environ.get('LOCPIR_B200_SMALL', '1')})")


if __name__ == "__main__":
    main()
