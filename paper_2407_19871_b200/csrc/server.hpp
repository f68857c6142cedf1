// server.hpp -- cross-session LocPIR query batcher over the C ABI.
//
// The reference server answers one QUERY at a time per session, evaluating loc_pir gate
// by gate (Server::handle_query, protocol.hpp:401-424).  Here sessions register their
// zero-sample sheet once (handle_zerosheet, protocol.hpp:373-398: services preprocessed
// into the session's own slots), QUERY payloads from any session queue up, and flush()
// evaluates all of them as ONE level-scheduled program -- every query reads its own
// session's service slots -- then packs RESPONSE payloads per ticket.  Boundaries are the
// server's plaintext boxes: trivial words in the pool, or constant-folded (flagged mode).
// Pure host C++ layered on the public entry points; no networking.
#pragma once
#include <cstdint>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/locpir_b200.h"
#include "circuits.hpp"

struct locpir_b200_server {
    locpir_b200_ctx* ctx = nullptr;
    uint32_t R = 0, l = 0, m = 0, max_sessions = 0, n = 0;
    int folded = 0;
    std::vector<int64_t> boxes;      // [R][4] signed grid values
    std::vector<uint64_t> services;  // [R] service values (the server's dataset)
    uint32_t base = 0;  // first pool slot the server owns (locpir_b200_server_create_at)
    uint32_t bnd_first = 0, svc_area = 0, flush_first = 0;
    std::vector<uint8_t> open;       // per session slot block
    struct Pending {
        uint64_t ticket;
        uint32_t session;
        std::vector<uint8_t> payload;
    };
    std::vector<Pending> pending;
    std::unordered_map<uint64_t, std::vector<uint8_t>> responses;
    uint64_t next_ticket = 1;
    std::string err;
};

namespace lpb {

inline void srv_ck(locpir_b200_server* s, int rc)
{
    if (rc == LOCPIR_B200_OK)
        return;
    const std::string msg = locpir_b200_last_error(s->ctx);
    if (rc == LOCPIR_B200_EINVAL)
        throw std::invalid_argument(msg);
    if (rc == LOCPIR_B200_ELOGIC)
        throw std::logic_error(msg);
    throw std::runtime_error(msg);
}

inline uint32_t srv_svc_first(const locpir_b200_server* s, uint32_t session)
{
    return s->svc_area + session * s->R * s->m;
}

// Bits of the l-bit two's-complement grid value v, LSB first (codec.hpp:50-86).
inline uint32_t grid_bit(int64_t v, uint32_t i) { return (uint32_t)(((uint64_t)v >> i) & 1u); }

inline void srv_init(locpir_b200_server* s)
{
    // pool from `base`: [R*4*l trivial boundary words][max_sessions * R*m service slots]
    // [flush area]
    s->bnd_first = s->base;
    s->svc_area = s->base + (s->folded ? 0 : s->R * 4 * s->l);
    s->flush_first = s->svc_area + s->max_sessions * s->R * s->m;
    srv_ck(s, locpir_b200_pool_reserve(s->ctx, s->flush_first));
    if (!s->folded) {  // dataset.hpp:250-253: boundaries as trivial words
        std::vector<locpir_b200_gate_op> ops;
        for (uint32_t r = 0; r < s->R; r++)
            for (uint32_t k = 0; k < 4; k++)
                for (uint32_t i = 0; i < s->l; i++)
                    ops.push_back({LOCPIR_B200_CONST, grid_bit(s->boxes[r * 4 + k], i), 0xFFFFFFFFu,
                                   0xFFFFFFFFu, s->bnd_first + (r * 4 + k) * s->l + i});
        srv_ck(s, locpir_b200_run(s->ctx, ops.data(), ops.size()));
    }
    s->open.assign(s->max_sessions, 0);
}

inline uint32_t srv_open(locpir_b200_server* s, const uint8_t* sheet, uint64_t len)
{
    uint32_t id = 0;
    while (id < s->max_sessions && s->open[id])
        id++;
    if (id == s->max_sessions)
        throw std::logic_error("no free session slot (max_sessions reached)");
    const uint64_t want = (uint64_t)s->R * s->m * 4ull * (s->n + 1);
    if (len != want)  // handle_zerosheet (protocol.hpp:380-385)
        throw std::invalid_argument("sheet payload is " + std::to_string(len) + " bytes, expected " +
                                    std::to_string(want));
    srv_ck(s, locpir_b200_pool_load_zero_sheet(s->ctx, sheet, len, s->R, s->m, s->services.data(),
                                               srv_svc_first(s, id)));
    s->open[id] = 1;
    return id;
}

inline uint64_t srv_submit(locpir_b200_server* s, uint32_t session, const uint8_t* q, uint64_t len)
{
    if (session >= s->max_sessions || !s->open[session])
        throw std::logic_error("QUERY before ZEROSHEET");  // protocol.hpp:403-404
    locpir_b200_params p{};
    p.n = s->n;
    char msg[256];
    if (locpir_b200_check_query_payload(&p, q, len, s->l, msg, sizeof msg) != LOCPIR_B200_OK)
        throw std::invalid_argument(msg);
    const uint64_t t = s->next_ticket++;
    s->pending.push_back({t, session, std::vector<uint8_t>(q, q + len)});
    return t;
}

inline uint64_t srv_flush(locpir_b200_server* s)
{
    const uint32_t Q = (uint32_t)s->pending.size();
    if (!Q)
        return 0;
    const uint32_t R = s->R, l = s->l, m = s->m;
    const uint32_t x0 = s->flush_first, y0 = x0 + Q * l, out0 = y0 + Q * l, scr = out0 + Q * m;
    const uint64_t need = (uint64_t)scr + (s->folded ? loc_pir_folded_scratch(Q, R, l, m)
                                                     : loc_pir_scratch(Q, R, l, m));
    srv_ck(s, locpir_b200_pool_reserve(s->ctx, need));
    std::vector<uint8_t> bytes;
    std::vector<uint64_t> offs{0};
    std::vector<uint32_t> xf(Q), yf(Q), xs((size_t)Q * l), ys((size_t)Q * l), outs((size_t)Q * m),
        of(Q);
    for (uint32_t q = 0; q < Q; q++) {
        bytes.insert(bytes.end(), s->pending[q].payload.begin(), s->pending[q].payload.end());
        offs.push_back(bytes.size());
        xf[q] = x0 + q * l;
        yf[q] = y0 + q * l;
        of[q] = out0 + q * m;
        for (uint32_t i = 0; i < l; i++) {
            xs[(size_t)q * l + i] = xf[q] + i;
            ys[(size_t)q * l + i] = yf[q] + i;
        }
        for (uint32_t j = 0; j < m; j++)
            outs[(size_t)q * m + j] = of[q] + j;
    }
    srv_ck(s, locpir_b200_pool_load_queries(s->ctx, bytes.data(), offs.data(), Q, l, xf.data(), yf.data()));
    std::vector<uint32_t> sess(Q);
    for (uint32_t q = 0; q < Q; q++)
        sess[q] = srv_svc_first(s, s->pending[q].session);
    auto svc = [&](uint32_t q, uint32_t r, uint32_t j) { return sess[q] + r * m + j; };
    std::vector<locpir_b200_gate_op> ops;
    if (s->folded) {
        emit_loc_pir_folded_fn(ops, Q, R, l, m, xs.data(), ys.data(), s->boxes.data(), svc,
                               outs.data(), scr, 1);
    } else {
        std::vector<uint32_t> bnd((size_t)R * 4 * l);
        for (size_t i = 0; i < bnd.size(); i++)
            bnd[i] = s->bnd_first + (uint32_t)i;
        emit_loc_pir_fn(ops, Q, R, l, m, xs.data(), ys.data(), bnd.data(), svc, outs.data(), scr, 1);
    }
    srv_ck(s, locpir_b200_run(s->ctx, ops.data(), ops.size()));
    const uint64_t S = 4ull * (s->n + 1);
    std::vector<uint8_t> resp((size_t)Q * m * S);
    srv_ck(s, locpir_b200_pool_store_responses(s->ctx, of.data(), Q, m, resp.data()));
    for (uint32_t q = 0; q < Q; q++)
        s->responses[s->pending[q].ticket] =
            std::vector<uint8_t>(resp.begin() + (size_t)q * m * S, resp.begin() + (size_t)(q + 1) * m * S);
    s->pending.clear();
    return Q;
}

template <class F>
inline int srv_guard(locpir_b200_server* s, F&& f)
{
    if (!s)
        return LOCPIR_B200_EINVAL;
    try {
        f();
        s->err.clear();
        return LOCPIR_B200_OK;
    } catch (const std::invalid_argument& e) {
        s->err = e.what();
        return LOCPIR_B200_EINVAL;
    } catch (const std::logic_error& e) {
        s->err = e.what();
        return LOCPIR_B200_ELOGIC;
    } catch (const std::bad_alloc&) {
        s->err = "out of memory";
        return LOCPIR_B200_ENOMEM;
    } catch (const std::exception& e) {
        s->err = e.what();
        return LOCPIR_B200_ECUDA;
    }
}

}  // namespace lpb
