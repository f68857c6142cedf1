"""Cross-session batcher (csrc/server.hpp): several sessions, each with its
own zero-sample sheet, submit QUERY payloads; one flush answers all of them in a single
batched program and the RESPONSE payloads decrypt to the reference's expected 9-city
answers (acceptance.cpp:180-237).  Error paths follow protocol.hpp:373-424."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _decrypt(resp: bytes, key, m):
    rows = np.frombuffer(resp, "<u4").reshape(m, -1)
    return sum(O.decrypt_bit(r, key) << j for j, r in enumerate(rows))


@pytest.mark.parametrize("level,folded", [(128, False), (128, True), (80, False)])
def test_sessions_batched_city_table(golden, level, folded):
    from test_wire import query_payload, zero_sheet_payload
    from paper_2407_19871_b200 import ClientKeys, Context, TfheParams
    from paper_2407_19871_b200.engine import InvalidArgument, LogicError
    from paper_2407_19871_b200.server import BatchingServer
    p = TfheParams(level)
    keys = ClientKeys(p, 41)
    ctx = Context(p, 0)
    ctx.upload_keys(keys.bk, keys.ksk)
    key = O.keygen_bits(p.n, 41)
    alpha = 2.0 ** -15 if level == 128 else 2.44e-5
    l, m = 16, golden["city_service_bits"][0]
    boxes = np.array(golden["city_boxes_grid_x1_x2_y1_y2_int32"], np.uint32).view(np.int32).reshape(-1, 4)
    R = boxes.shape[0]
    srv = BatchingServer(ctx, boxes, golden["city_services"], l, m, max_sessions=4, folded=folded)
    with pytest.raises(LogicError, match="QUERY before ZEROSHEET"):
        srv.submit(0, b"\x10")
    sessions = []
    for s in range(3):
        sheet, _ = zero_sheet_payload(key, O.NoiseSampler(300 + s, alpha), R, m)
        sessions.append(srv.open_session(sheet))
    with pytest.raises(InvalidArgument, match="sheet payload is"):
        srv.open_session(sheet[:-1])
    qs = np.array(golden["city_queries_grid_xy_int32"], np.uint32).view(np.int32).reshape(-1, 2)
    smp = O.NoiseSampler(400, alpha)
    tickets = []
    for i, (gx, gy) in enumerate(qs):
        tickets.append(srv.submit(sessions[i % 3], query_payload(key, smp, gx, gy, l)[0]))
    with pytest.raises(InvalidArgument, match="does not match negotiated format"):
        srv.submit(sessions[0], query_payload(key, smp, 1, 2, 13)[0])
    assert srv.pending == len(qs)
    with pytest.raises(LogicError, match="not flushed"):
        srv.take_response(tickets[0])
    assert srv.flush() == len(qs)
    got = [_decrypt(srv.take_response(t), key, m) for t in tickets]
    assert got == golden["city_expected"]
    # a second round on the same sessions reuses their service slots
    t2 = srv.submit(sessions[2], query_payload(key, smp, qs[0][0], qs[0][1], l)[0])
    srv.flush()
    assert _decrypt(srv.take_response(t2), key, m) == golden["city_expected"][0]
    srv.close_session(sessions[1])
    with pytest.raises(LogicError):
        srv.submit(sessions[1], query_payload(key, smp, 1, 2, l)[0])
    srv.close()
    ctx.close()


def test_server_and_engine_share_a_context(golden):
    """a GateEngine and a BatchingServer on one context no longer share slots.
    The engine caps itself below reserve_server_tail(); the server owns the tail; engine
    values made before the server survive a flush; a raw call into the tail is refused."""
    from test_wire import query_payload, zero_sheet_payload
    from paper_2407_19871_b200 import ClientKeys, Context, TfheParams
    from paper_2407_19871_b200.engine import GateEngine, InvalidArgument
    from paper_2407_19871_b200.server import BatchingServer
    p = TfheParams(128)
    keys = ClientKeys(p, 41)
    ctx = Context(p, 0)
    ctx.upload_keys(keys.bk, keys.ksk)
    eng = GateEngine(ctx, keys, seed=5)
    one = eng.hom_xor(eng.encrypt(1), eng.encrypt(0))
    zero = eng.hom_and(eng.encrypt(1), eng.encrypt(0))
    base = eng.reserve_server_tail(headroom=64)
    key = O.keygen_bits(p.n, 41)
    l, m = 16, golden["city_service_bits"][0]
    boxes = np.array(golden["city_boxes_grid_x1_x2_y1_y2_int32"], np.uint32).view(np.int32).reshape(-1, 4)
    srv = BatchingServer(ctx, boxes, golden["city_services"], l, m, max_sessions=1, base_slot=base)
    sheet, _ = zero_sheet_payload(key, O.NoiseSampler(300, 2.0 ** -15), boxes.shape[0], m)
    sid = srv.open_session(sheet)
    qs = np.array(golden["city_queries_grid_xy_int32"], np.uint32).view(np.int32).reshape(-1, 2)
    t = srv.submit(sid, query_payload(key, O.NoiseSampler(400, 2.0 ** -15), qs[0][0], qs[0][1], l)[0])
    srv.flush()
    assert _decrypt(srv.take_response(t), key, m) == golden["city_expected"][0]
    assert eng.decrypt(one) == 1 and eng.decrypt(zero) == 0
    assert eng.decrypt(eng.hom_or(one, zero)) == 1
    with pytest.raises(InvalidArgument, match="owned by the batching server"):
        ctx.h2d(base, keys.encrypt_bits(np.ones(1, np.uint8), 1))
    srv.close()
    ctx.h2d(base, keys.encrypt_bits(np.ones(1, np.uint8), 1))  # free again
    eng.reset_slots()
    with pytest.raises(InvalidArgument, match="predates reset_slots"):
        eng.decrypt(one)
    ctx.close()
