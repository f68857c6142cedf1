"""Wire payloads <-> device pool.  The reference's QUERY / ZEROSHEET /
RESPONSE byte formats are pinned by digests of payloads the unmodified reference made
(tests/golden/ref_vectors.json, wire_*); the B200 unpack/pack path must land exactly the
samples those bytes carry, and the 9-city table must come back through the wire
(acceptance.cpp:180-237, test_protocol.cpp:97-191)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_19871_b200.circuits import FixedPointFormat, PlainWord
from paper_2407_19871_b200.engine import InvalidArgument, TfheParams, check_query_payload


def fnv1a64(b: bytes):
    h = 1469598103934665603
    for c in b:
        h = ((h ^ c) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return [h & 0xFFFFFFFF, h >> 32]


def grid_bits(v: int, l: int):
    return PlainWord.from_integer(int(v), FixedPointFormat(9, l - 9)).bits


def query_payload(key, sampler, gx: int, gy: int, l: int):
    """protocol.hpp:185-193: two framed words (u8 l + l raw samples), lat then lon."""
    out = b""
    samples = []
    for g in (gx, gy):
        cts = [O.encrypt_bit(b, key, sampler) for b in grid_bits(g, l)]
        samples.append(np.stack(cts))
        out += bytes([l]) + np.stack(cts).astype("<u4").tobytes()
    return out, samples


def zero_sheet_payload(key, sampler, regions, bits):
    cts = np.stack([O.encrypt_torus(0, key, sampler) for _ in range(regions * bits)])
    return cts.astype("<u4").tobytes(), cts


def preprocess(cts, values, bits):
    out = cts.copy()
    for i in range(out.shape[0]):
        r, j = divmod(i, bits)
        out[i, -1] = (int(out[i, -1]) + (0x20000000 if (values[r] >> j) & 1 else 0xE0000000)) & 0xFFFFFFFF
    return out


@pytest.fixture(scope="module")
def ref_wire(golden):
    key = O.keygen_bits(630, 12)  # reference sec128: n = 630, sigma = 2^-13.8 (torus.hpp:77)
    ln, gx, gy = golden["wire_query_len_lat_lon_grid"]
    q, qs = query_payload(key, O.NoiseSampler(17, 2.0 ** -13.8), np.int32(np.uint32(gx)),
                          np.int32(np.uint32(gy)), 16)
    zs, zc = zero_sheet_payload(key, O.NoiseSampler(18, 2.0 ** -13.8), 3, 4)
    return dict(key=key, query=q, query_samples=qs, sheet=zs, sheet_cts=zc)


def test_client_payloads_match_reference_bytes(golden, ref_wire):
    assert len(ref_wire["query"]) == golden["wire_query_len_lat_lon_grid"][0]
    assert fnv1a64(ref_wire["query"]) == golden["wire_query_fnv1a64"]
    assert len(ref_wire["sheet"]) == golden["wire_zerosheet_len"][0]
    assert fnv1a64(ref_wire["sheet"]) == golden["wire_zerosheet_fnv1a64"]
    pre = preprocess(ref_wire["sheet_cts"], [5, 9, 14], 4)
    assert fnv1a64(pre.astype("<u4").tobytes()) == golden["wire_services_5_9_14_fnv1a64"]


def test_query_framing_checks_mirror_the_reference(ref_wire):
    p = TfheParams(128)
    q = ref_wire["query"]
    check_query_payload(p, q, 16)
    cases = [
        (q, 13, "cipher word length 16 does not match negotiated format l=13"),
        (q[:-3], 16, "truncated input: need 4 bytes, have 1"),
        (q + b"\0\0", 16, "trailing bytes: 2"),
        (b"", 16, "truncated input: need 1 bytes, have 0"),
        (q[: len(q) // 2], 16, "truncated input: need 1 bytes, have 0"),
        (q[: len(q) // 2] + b"\x0f", 16,
         "cipher word length 15 does not match negotiated format l=16"),
    ]
    for payload, l, msg in cases:
        with pytest.raises(InvalidArgument, match=msg):
            check_query_payload(p, payload, l)


@pytest.mark.gpu
def test_wire_payloads_through_the_pool(golden, ref_wire):
    from paper_2407_19871_b200 import Context
    p = TfheParams(128)
    ctx = Context(p, 0)
    ctx.pool_reserve(200)
    # three copies of the reference query at different offsets, slots interleaved
    ctx.load_queries([ref_wire["query"]] * 3, 16, [0, 40, 80], [20, 60, 100])
    xs, ys = ref_wire["query_samples"]
    for base in (0, 40, 80):
        assert np.array_equal(ctx.d2h(base, 16), xs)
        assert np.array_equal(ctx.d2h(base + 20, 16), ys)
    ctx.load_zero_sheet(ref_wire["sheet"], 3, 4, [5, 9, 14], 150)
    pre = ctx.d2h(150, 12)
    assert fnv1a64(pre.astype("<u4").tobytes()) == golden["wire_services_5_9_14_fnv1a64"]
    resp = ctx.store_responses([154, 150], 4)
    assert resp[0] == pre[4:8].astype("<u4").tobytes()
    got = sum(O.decrypt_bit(r, ref_wire["key"]) << j
              for j, r in enumerate(np.frombuffer(resp[0], "<u4").reshape(4, -1)))
    assert got == golden["wire_response_region1_value"][0] == 9
    with pytest.raises(InvalidArgument, match="does not match negotiated format"):
        ctx.load_queries([ref_wire["query"]], 12, [0], [20])
    with pytest.raises(InvalidArgument, match="zero-sample sheet payload is"):
        ctx.load_zero_sheet(ref_wire["sheet"][:-4], 3, 4, [5, 9, 14], 150)
    with pytest.raises(InvalidArgument, match="does not fit in 4 bits"):
        ctx.load_zero_sheet(ref_wire["sheet"], 3, 4, [5, 99, 14], 150)
    ctx.close()


@pytest.mark.gpu
@pytest.mark.parametrize("level", [80, 128])
def test_city_table_through_the_wire(golden, level):
    """Client payload bytes in, RESPONSE bytes out: ZEROSHEET -> preprocessed services,
    trivial boundary words, QUERY payloads, batched loc_pir, RESPONSE pack; the client
    decrypts the reference's own expected answers (acceptance.cpp:180-237)."""
    from paper_2407_19871_b200 import Context, _abi
    from paper_2407_19871_b200.engine import loc_pir_program
    p = TfheParams(level)
    n = p.n
    key = O.keygen_bits(n, 77)
    ctx = Context(p, 0)
    keys = __import__("paper_2407_19871_b200").ClientKeys(p, 77)
    ctx.upload_keys(keys.bk, keys.ksk)
    l, m = 16, golden["city_service_bits"][0]
    boxes = np.array(golden["city_boxes_grid_x1_x2_y1_y2_int32"], np.uint32).view(np.int32).reshape(-1, 4)
    R = boxes.shape[0]
    qs = np.array(golden["city_queries_grid_xy_int32"], np.uint32).view(np.int32).reshape(-1, 2)
    Q = qs.shape[0]
    alpha = 2.0 ** -15 if level == 128 else 2.44e-5
    s = O.NoiseSampler(99, alpha)
    payloads = [query_payload(key, s, gx, gy, l)[0] for gx, gy in qs]
    sheet, _ = zero_sheet_payload(key, s, R, m)
    x = np.arange(Q * l, dtype=np.uint32).reshape(Q, l)
    y = Q * l + np.arange(Q * l, dtype=np.uint32).reshape(Q, l)
    bnd = 2 * Q * l + np.arange(R * 4 * l, dtype=np.uint32).reshape(R, 4, l)
    svc = int(bnd.max()) + 1 + np.arange(R * m, dtype=np.uint32).reshape(R, m)
    out = int(svc.max()) + 1 + np.arange(Q * m, dtype=np.uint32).reshape(Q, m)
    scratch = int(out.max()) + 1
    ctx.pool_reserve(scratch + _abi.lib().locpir_b200_loc_pir_scratch(Q, R, l, m))
    ctx.run([(_abi.CONST, int(b), 0, 0, int(bnd[r, k, i]))
             for r in range(R) for k in range(4) for i, b in enumerate(grid_bits(boxes[r, k], l))])
    ctx.load_zero_sheet(sheet, R, m, golden["city_services"], int(svc.min()))
    ctx.load_queries(payloads, l, x[:, 0], y[:, 0])
    ops = loc_pir_program(Q, R, l, m, x, y, bnd, svc, out, scratch)
    prog = ctx.program(ops)
    prog.launch()
    resp = ctx.store_responses(out[:, 0], m)
    got = [sum(O.decrypt_bit(r, key) << j for j, r in enumerate(np.frombuffer(b, "<u4").reshape(m, -1)))
           for b in resp]
    assert got == golden["city_expected"]
    prog.close()
    ctx.close()
