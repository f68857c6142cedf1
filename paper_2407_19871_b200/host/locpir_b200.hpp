// locpir_b200.hpp -- header-only C++ mirror of the reference engine boundary over
// the B200 C ABI (include/locpir_b200.h).
//
// Mirrors locpir::GateEngine (/root/reference/proj/include/locpir/gate_engine.hpp:
// 130-336): same method names, argument meaning and exception types
// (std::invalid_argument for foreign bits / bad arguments, std::logic_error for
// missing keys).  The engine kind is "tfhe-b200"; parse_engine_kind("tfhe") still
// throws (test_gate_engine.cpp:154).  Gates can run eagerly (one gate per launch,
// like the reference) or be recorded between begin_batch() and flush(), in which
// case the circuit scheduler runs every independent gate of a level as one batch.
// The circuits (hom_less, hom_less_equal, mask_service, xor_sum_services, loc_pir)
// follow circuits.hpp:187-324 gate for gate.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "../../include/locpir_b200.h"

namespace locpir_b200 {

enum class EngineKind : uint8_t { Clear = 0, TlweOracle = 1, TfheB200 = 2 };

inline EngineKind parse_engine_kind(std::string_view s)
{
    if (s == "clear")
        return EngineKind::Clear;
    if (s == "tlwe-oracle")
        return EngineKind::TlweOracle;
    if (s == "tfhe-b200")
        return EngineKind::TfheB200;
    throw std::invalid_argument("unknown engine \"" + std::string(s) +
                                "\" (expected clear, tlwe-oracle or tfhe-b200)");
}

inline void check(int rc, const locpir_b200_ctx* ctx = nullptr)
{
    if (rc == LOCPIR_B200_OK)
        return;
    const std::string msg = ctx ? locpir_b200_last_error(ctx) : "";
    if (rc == LOCPIR_B200_EINVAL)
        throw std::invalid_argument(msg.empty() ? "invalid argument" : msg);
    if (rc == LOCPIR_B200_ELOGIC)
        throw std::logic_error(msg.empty() ? "logic error" : msg);
    throw std::runtime_error("locpir_b200: " + (msg.empty() ? std::to_string(rc) : msg));
}

struct Params {
    locpir_b200_params c{};
    static Params tfhe(int bits)
    {
        Params p;
        check(locpir_b200_params_default(bits, &p.c));
        return p;
    }
    static Params tfhe80() { return tfhe(80); }
    static Params tfhe128() { return tfhe(128); }
    uint32_t n() const { return c.n; }
    size_t sample_words() const { return c.n + 1; }
};

// Client-side secrets and the public evaluation keys, all from one seed.
struct ClientKeys {
    Params params;
    std::vector<uint8_t> lwe_key, trlwe_key;
    std::vector<uint32_t> bk, ksk;

    ClientKeys(Params p, uint64_t seed, bool evaluation_keys = true) : params(p)
    {
        lwe_key.resize(p.c.n);
        trlwe_key.resize(p.c.N);
        if (evaluation_keys) {
            bk.resize(locpir_b200_bk_words(&p.c));
            ksk.resize(locpir_b200_ksk_words(&p.c));
        }
        check(locpir_b200_keygen(&p.c, seed, lwe_key.data(), trlwe_key.data(),
                                 evaluation_keys ? bk.data() : nullptr,
                                 evaluation_keys ? ksk.data() : nullptr));
    }

    std::vector<uint32_t> encrypt(const std::vector<uint8_t>& bits, uint64_t seed) const
    {
        std::vector<uint32_t> out(bits.size() * params.sample_words());
        check(locpir_b200_encrypt_bits(&params.c, lwe_key.data(), seed, bits.data(),
                                       bits.size(), out.data()));
        return out;
    }
    std::vector<uint8_t> decrypt(const std::vector<uint32_t>& cts) const
    {
        std::vector<uint8_t> out(cts.size() / params.sample_words());
        check(locpir_b200_decrypt_bits(&params.c, lwe_key.data(), cts.data(), out.size(),
                                       out.data()));
        return out;
    }
};

// One encrypted bit: a slot of the engine's device pool (gate_engine.hpp:81-109).
class CipherBit {
public:
    CipherBit() = default;
    EngineKind kind() const { return EngineKind::TfheB200; }
    uint32_t slot() const { return slot_; }

private:
    friend class GateEngine;
    CipherBit(uint64_t engine, uint64_t epoch, uint32_t slot) : engine_(engine), epoch_(epoch), slot_(slot) {}
    uint64_t engine_ = 0;
    uint64_t epoch_ = 0;  // slot arena generation (GateEngine::reset_slots)
    uint32_t slot_ = 0xFFFFFFFFu;
};

struct GateCounterSnapshot {
    uint64_t and_gates = 0, or_gates = 0, xor_gates = 0, xnor_gates = 0, not_gates = 0,
             mux_gates = 0, nand_gates = 0, nor_gates = 0;
    uint64_t other_units = 0;  // flagged single-bootstrap gates outside the reference set (MAJ, XOR3)
    uint64_t bootstrap_units() const  // gate_engine.hpp:44-48 (+ NAND/NOR)
    {
        return and_gates + or_gates + xor_gates + xnor_gates + nand_gates + nor_gates +
               2 * mux_gates + other_units;
    }
    std::map<std::string, uint64_t> as_map() const
    {
        return {{"and", and_gates},   {"or", or_gates},     {"xor", xor_gates},
                {"xnor", xnor_gates}, {"not", not_gates},   {"mux", mux_gates},
                {"nand", nand_gates}, {"nor", nor_gates},   {"bootstrap_units", bootstrap_units()}};
    }
};

class GateEngine {
public:
    static GateEngine make_b200(const ClientKeys& keys, uint64_t seed, int device = 0,
                                uint64_t pool_slots = 1 << 16)
    {
        return GateEngine(keys, seed, device, pool_slots);
    }

    EngineKind kind() const { return EngineKind::TfheB200; }
    // Deterministic bootstrap: forks share the recorder (one context, every mutating call
    // under the State mutex), so gates on distinct bits may be recorded from concurrent
    // forks as the reference's circuits do (gate_engine.hpp:128-129).
    GateEngine fork(uint64_t /*lane*/) const { return *this; }
    uint64_t acquire_fork_block() const { return st_->fork_blocks.fetch_add(1); }
    const Params& params() const { return st_->keys.params; }
    const std::vector<uint8_t>& secret_key() const { return st_->keys.lwe_key; }

    GateCounterSnapshot counters() const
    {
        const_cast<GateEngine*>(this)->flush();
        uint64_t c[9];
        check(locpir_b200_counters(st_->ctx, c), st_->ctx);
        GateCounterSnapshot snap{c[0], c[1], c[2], c[3], c[4], c[5], c[6], c[7]};
        snap.other_units = c[8] - snap.bootstrap_units();  // the library's unit total
        return snap;
    }
    void reset_counters() { check(locpir_b200_counters_reset(st_->ctx), st_->ctx); }

    // -- client-side helpers (tests, demos) ---------------------------------
    CipherBit constant(bool b) { return emit(LOCPIR_B200_CONST, b ? 1u : 0u); }
    CipherBit encrypt(bool b) { return encrypt_many({static_cast<uint8_t>(b)})[0]; }
    std::vector<CipherBit> encrypt_many(const std::vector<uint8_t>& bits)
    {
        std::lock_guard<std::recursive_mutex> g(st_->mu);
        flush();
        const auto cts = st_->keys.encrypt(bits, st_->seed + st_->enc_calls++);
        const uint32_t first = alloc(bits.size());
        check(locpir_b200_pool_h2d(st_->ctx, first, bits.size(), cts.data()), st_->ctx);
        std::vector<CipherBit> out;
        for (uint32_t i = 0; i < bits.size(); i++)
            out.push_back(CipherBit(st_->id, st_->epoch, first + i));
        return out;
    }
    std::vector<uint32_t> sample(const CipherBit& c)
    {
        std::lock_guard<std::recursive_mutex> g(st_->mu);
        flush();
        std::vector<uint32_t> out(params().sample_words());
        check(locpir_b200_pool_d2h(st_->ctx, slot(c), 1, out.data()), st_->ctx);
        return out;
    }
    bool decrypt(const CipherBit& c) { return st_->keys.decrypt(sample(c))[0] != 0; }

    // -- gates (gate_engine.hpp:196-269) ---------------------------------------
    CipherBit hom_and(const CipherBit& a, const CipherBit& b) { return emit2(LOCPIR_B200_AND, a, b); }
    CipherBit hom_or(const CipherBit& a, const CipherBit& b) { return emit2(LOCPIR_B200_OR, a, b); }
    CipherBit hom_xor(const CipherBit& a, const CipherBit& b) { return emit2(LOCPIR_B200_XOR, a, b); }
    CipherBit hom_xnor(const CipherBit& a, const CipherBit& b) { return emit2(LOCPIR_B200_XNOR, a, b); }
    CipherBit hom_nand(const CipherBit& a, const CipherBit& b) { return emit2(LOCPIR_B200_NAND, a, b); }
    CipherBit hom_nor(const CipherBit& a, const CipherBit& b) { return emit2(LOCPIR_B200_NOR, a, b); }
    CipherBit hom_not(const CipherBit& a) { return emit(LOCPIR_B200_NOT, slot(a)); }
    CipherBit hom_mux(const CipherBit& s, const CipherBit& a, const CipherBit& b)
    {
        return emit(LOCPIR_B200_MUX, slot(s), slot(a), slot(b));
    }
    // 3-input majority in ONE bootstrap (flagged comparator mode; not in the reference)
    CipherBit hom_maj(const CipherBit& a, const CipherBit& b, const CipherBit& c)
    {
        return emit(LOCPIR_B200_MAJ, slot(a), slot(b), slot(c));
    }
    // a ^ b ^ c in ONE bootstrap (flagged ternary XOR trees; not in the reference)
    CipherBit hom_xor3(const CipherBit& a, const CipherBit& b, const CipherBit& c)
    {
        return emit(LOCPIR_B200_XOR3, slot(a), slot(b), slot(c));
    }

    // the context behind this engine (for BatchingServer and other C-ABI users)
    locpir_b200_ctx* native()
    {
        flush();
        return st_->ctx;
    }

    // Slot arena.  Every gate output owns one pool slot (n+1 words) until reset_slots():
    // a long-running caller (e.g. one loc_pir per query) resets between independent
    // evaluations.  Bits from before a reset are rejected (invalid_argument), never aliased.
    void reset_slots()
    {
        std::lock_guard<std::recursive_mutex> g(st_->mu);
        flush();
        st_->next_slot = 0;
        st_->epoch++;
    }
    uint64_t slots_in_use() const { return st_->next_slot; }

    // Caps this engine's slots below the returned base and hands [base, ...) to a
    // BatchingServer on the same context (locpir_b200_server_create_at).  `headroom`
    // more slots stay available to the engine.
    uint64_t reserve_server_tail(uint64_t headroom = 1u << 16)
    {
        std::lock_guard<std::recursive_mutex> g(st_->mu);
        flush();
        st_->limit = std::min<uint64_t>(st_->limit, st_->next_slot + headroom);
        return st_->limit;
    }

    // -- level batching ---------------------------------------------------------
    void begin_batch()
    {
        std::lock_guard<std::recursive_mutex> g(st_->mu);
        st_->batching++;
    }
    void end_batch()
    {
        std::lock_guard<std::recursive_mutex> g(st_->mu);
        if (st_->batching > 0 && --st_->batching == 0)
            flush();
    }
    void flush()
    {
        std::lock_guard<std::recursive_mutex> g(st_->mu);
        if (st_->pending.empty())
            return;
        std::vector<locpir_b200_gate_op> ops;
        ops.swap(st_->pending);
        check(locpir_b200_run(st_->ctx, ops.data(), ops.size()), st_->ctx);
    }

private:
    struct State {
        ClientKeys keys;
        locpir_b200_ctx* ctx = nullptr;
        uint64_t id = 0, seed = 0, enc_calls = 0;
        uint64_t next_slot = 0, epoch = 0;
        uint64_t limit = 0xFFFFFFF0ull;  // first slot the engine may not use
        uint64_t capacity = 0;
        int batching = 0;
        std::atomic<uint64_t> fork_blocks{0};
        std::recursive_mutex mu;
        std::vector<locpir_b200_gate_op> pending;
        explicit State(const ClientKeys& k) : keys(k) {}
        ~State()
        {
            if (ctx)
                locpir_b200_ctx_destroy(ctx);
        }
    };

    GateEngine(const ClientKeys& keys, uint64_t seed, int device, uint64_t pool_slots)
        : st_(std::make_shared<State>(keys))
    {
        static uint64_t ids = 0;
        st_->id = ++ids;
        st_->seed = seed;
        check(locpir_b200_ctx_create(&keys.params.c, device, nullptr, &st_->ctx));
        if (keys.bk.empty())
            throw std::logic_error("the engine needs the bootstrapping and key-switching keys");
        check(locpir_b200_upload_keys(st_->ctx, keys.bk.data(), keys.ksk.data(), 0), st_->ctx);
        grow(pool_slots);
    }

    void grow(uint64_t want)
    {
        check(locpir_b200_pool_reserve(st_->ctx, want), st_->ctx);
        st_->capacity = locpir_b200_pool_capacity(st_->ctx);
    }
    uint32_t alloc(uint64_t k)
    {
        const uint64_t s = st_->next_slot;
        if (s + k > st_->limit)
            throw std::logic_error("engine slot range exhausted at slot " + std::to_string(s) +
                                   " (reset_slots() between evaluations, or a server owns the "
                                   "pool tail)");
        st_->next_slot += k;
        if (st_->next_slot > st_->capacity) {
            flush();
            grow(std::min<uint64_t>(st_->limit, std::max<uint64_t>(st_->next_slot, 2 * st_->capacity)));
        }
        return static_cast<uint32_t>(s);
    }
    uint32_t slot(const CipherBit& c) const
    {
        if (c.engine_ != st_->id)
            throw std::invalid_argument("cipher bit belongs to a different engine");
        if (c.epoch_ != st_->epoch)
            throw std::invalid_argument("cipher bit predates reset_slots()");
        return c.slot_;
    }
    CipherBit emit2(uint32_t kind, const CipherBit& a, const CipherBit& b)
    {
        return emit(kind, slot(a), slot(b));
    }
    CipherBit emit(uint32_t kind, uint32_t a, uint32_t b = 0xFFFFFFFFu, uint32_t c = 0xFFFFFFFFu)
    {
        std::lock_guard<std::recursive_mutex> g(st_->mu);
        const uint32_t out = alloc(1);
        st_->pending.push_back({kind, a, b, c, out});
        if (!st_->batching)
            flush();
        return CipherBit(st_->id, st_->epoch, out);
    }

    std::shared_ptr<State> st_;
};

// ---- circuits (circuits.hpp:187-324) -------------------------------------------
struct CipherWord {
    std::vector<CipherBit> bits;  // index 0 = LSB (codec.hpp:106-109)
    // FixedPointFormat (codec.hpp:16-30); int_bits = frac_bits = 0 leaves it unspecified
    // (then only the length is compared)
    uint8_t int_bits = 0, frac_bits = 0;
};

inline bool same_format(const CipherWord& a, const CipherWord& b)
{
    return a.bits.size() == b.bits.size() && a.int_bits == b.int_bits && a.frac_bits == b.frac_bits;
}

struct ServiceCiphertext {
    std::vector<CipherBit> bits;
};

struct EncodedRegion {
    CipherWord x1, x2, y1, y2;  // [x1, x2) x [y1, y2)
    ServiceCiphertext service;
    uint32_t region_id = 0;
};

struct BatchScope {
    GateEngine& e;
    explicit BatchScope(GateEngine& eng) : e(eng) { e.begin_batch(); }
    ~BatchScope() { e.end_batch(); }
};

inline CipherBit hom_less(const CipherWord& a, const CipherWord& b, GateEngine& e)
{
    if (!same_format(a, b))
        throw std::invalid_argument("comparator operands must share length and format");
    if (a.bits.empty())
        throw std::invalid_argument("comparator operands must be non-empty");
    BatchScope scope(e);
    const size_t l = a.bits.size();
    const CipherBit a_sign = e.hom_not(a.bits[l - 1]);
    const CipherBit b_sign = e.hom_not(b.bits[l - 1]);
    CipherBit t0 = e.constant(false);
    for (size_t i = 0; i < l; i++) {
        const CipherBit& ai = (i + 1 == l) ? a_sign : a.bits[i];
        const CipherBit& bi = (i + 1 == l) ? b_sign : b.bits[i];
        const CipherBit t1 = e.hom_xnor(ai, bi);
        t0 = e.hom_mux(t1, t0, bi);
    }
    return t0;
}

inline CipherBit hom_less_equal(const CipherWord& a, const CipherWord& b, GateEngine& e)
{
    BatchScope scope(e);
    return e.hom_not(hom_less(b, a, e));
}

inline ServiceCiphertext mask_service(const CipherBit& f, const ServiceCiphertext& s, GateEngine& e)
{
    BatchScope scope(e);
    ServiceCiphertext out;
    for (const CipherBit& b : s.bits)
        out.bits.push_back(e.hom_and(f, b));
    return out;
}

// N*m XOR units; tree = false is the reference chain (circuits.hpp:257-261).
inline ServiceCiphertext xor_sum_services(const std::vector<ServiceCiphertext>& in, GateEngine& e,
                                          bool tree = true)
{
    if (in.empty())
        return {};
    const size_t m = in[0].bits.size();
    for (const auto& s : in)
        if (s.bits.size() != m)
            throw std::invalid_argument("service ciphertexts must share bit-length");
    BatchScope scope(e);
    ServiceCiphertext out;
    for (size_t j = 0; j < m; j++) {
        CipherBit acc = e.constant(false);
        if (!tree) {
            for (const auto& s : in)
                acc = e.hom_xor(acc, s.bits[j]);
        } else {
            std::vector<CipherBit> lvl;
            for (const auto& s : in)
                lvl.push_back(s.bits[j]);
            while (lvl.size() > 1) {
                std::vector<CipherBit> nxt;
                for (size_t i = 0; i + 1 < lvl.size(); i += 2)
                    nxt.push_back(e.hom_xor(lvl[i], lvl[i + 1]));
                if (lvl.size() & 1)
                    nxt.push_back(lvl.back());
                lvl.swap(nxt);
            }
            acc = e.hom_xor(acc, lvl[0]);
        }
        out.bits.push_back(acc);
    }
    return out;
}

// Flagged comparator: a < b = borrow out of a' - b' with both sign bits flipped,
// borrow_{i+1} = MAJ(NOT a'_i, b'_i, borrow_i): l bootstraps instead of 3l.
inline CipherBit hom_less_maj(const CipherWord& a, const CipherWord& b, GateEngine& e)
{
    if (!same_format(a, b) || a.bits.empty())
        throw std::invalid_argument("comparator operands must share length and format");
    BatchScope scope(e);
    const size_t l = a.bits.size();
    CipherBit borrow = e.constant(false);
    for (size_t i = 0; i < l; i++) {
        const bool sign = i + 1 == l;
        const CipherBit na = sign ? a.bits[i] : e.hom_not(a.bits[i]);
        const CipherBit bi = sign ? e.hom_not(b.bits[i]) : b.bits[i];
        borrow = e.hom_maj(na, bi, borrow);
    }
    return borrow;
}

enum class Comparator { Reference, Majority };

inline ServiceCiphertext loc_pir(const CipherWord& x, const CipherWord& y,
                                 const std::vector<EncodedRegion>& regions, GateEngine& e,
                                 bool tree = true, Comparator cmp = Comparator::Reference)
{
    if (regions.empty())
        return {};
    // the reference's argument checks (circuits.hpp:283-292)
    if (!same_format(x, y))
        throw std::invalid_argument("coordinate words must share a format");
    const size_t m = regions[0].service.bits.size();
    for (const EncodedRegion& r : regions) {
        if (!same_format(r.x1, x) || !same_format(r.x2, x) || !same_format(r.y1, y) ||
            !same_format(r.y2, y))
            throw std::invalid_argument("region boundary format mismatch");
        if (r.service.bits.size() != m)
            throw std::invalid_argument("regions must share the service bit-length");
    }
    BatchScope scope(e);
    auto lt = [&](const CipherWord& a, const CipherWord& b) {
        return cmp == Comparator::Majority ? hom_less_maj(a, b, e) : hom_less(a, b, e);
    };
    std::vector<ServiceCiphertext> masked;
    for (const EncodedRegion& r : regions) {
        const CipherBit x_l = e.hom_not(lt(x, r.x1));
        const CipherBit x_r = lt(x, r.x2);
        const CipherBit y_l = e.hom_not(lt(y, r.y1));
        const CipherBit y_r = lt(y, r.y2);
        const CipherBit v1 = e.hom_and(x_l, x_r);
        const CipherBit v2 = e.hom_and(y_l, y_r);
        const CipherBit f = e.hom_and(v1, v2);
        masked.push_back(mask_service(f, r.service, e));
    }
    return xor_sum_services(masked, e, tree);
}

// ---- cross-session query batcher (csrc/server.hpp) ---------------------
// Server::handle_zerosheet / handle_query (protocol.hpp:373-424) without the transport:
// wire payloads in, RESPONSE payloads out, one batched program per flush().
class BatchingServer {
public:
    BatchingServer(GateEngine& eng, const std::vector<int64_t>& boxes /* [R][4] grid */,
                   const std::vector<uint64_t>& services, uint32_t l, uint32_t m,
                   uint32_t max_sessions = 64, bool folded = false)
        : m_(m), n_(eng.params().n())
    {
        if (boxes.size() != services.size() * 4)
            throw std::invalid_argument("one service value per box");
        // the server owns the pool tail from the engine's cap on (no shared slots)
        const uint64_t base = eng.reserve_server_tail();
        locpir_b200_ctx* c = eng.native();
        check(locpir_b200_server_create_at(c, base, boxes.data(), services.data(),
                                           (uint32_t)services.size(), l, m, max_sessions,
                                           folded ? 1 : 0, &s_),
              c);
    }
    ~BatchingServer() { locpir_b200_server_destroy(s_); }
    BatchingServer(const BatchingServer&) = delete;
    BatchingServer& operator=(const BatchingServer&) = delete;

    uint32_t open_session(const std::vector<uint8_t>& zero_sheet)
    {
        uint32_t id = 0;
        ck(locpir_b200_server_open_session(s_, zero_sheet.data(), zero_sheet.size(), &id));
        return id;
    }
    void close_session(uint32_t id) { ck(locpir_b200_server_close_session(s_, id)); }
    uint64_t submit(uint32_t session, const std::vector<uint8_t>& query)
    {
        uint64_t t = 0;
        ck(locpir_b200_server_submit(s_, session, query.data(), query.size(), &t));
        return t;
    }
    uint64_t pending() const { return locpir_b200_server_pending(s_); }
    uint64_t flush()
    {
        uint64_t n = 0;
        ck(locpir_b200_server_flush(s_, &n));
        return n;
    }
    std::vector<uint8_t> take_response(uint64_t ticket)
    {
        std::vector<uint8_t> out((size_t)m_ * 4 * (n_ + 1));
        ck(locpir_b200_server_take_response(s_, ticket, out.data(), out.size()));
        return out;
    }

private:
    void ck(int rc)
    {
        if (rc == LOCPIR_B200_OK)
            return;
        const std::string msg = locpir_b200_server_last_error(s_);
        if (rc == LOCPIR_B200_EINVAL)
            throw std::invalid_argument(msg);
        if (rc == LOCPIR_B200_ELOGIC)
            throw std::logic_error(msg);
        throw std::runtime_error(msg);
    }
    locpir_b200_server* s_ = nullptr;
    uint32_t m_, n_;
};

}  // namespace locpir_b200
