// integration/locpir/gate_engine.hpp -- drop-in replacement for the reference's
// locpir/gate_engine.hpp (/root/reference/proj/include/locpir/gate_engine.hpp:1-338)
// that adds the B200 engine kind "tfhe-b200" behind the same class interface.
//
// Put this directory ahead of the reference's include directory:
//     g++ -Iintegration -I<reference>/proj/include -Iinclude ... -llocpir_b200
// and the reference's UNMODIFIED callers -- circuits.hpp (hom_less, mask_service,
// xor_sum_services, loc_pir), codec.hpp (constant_word, encrypt_word, decrypt_word),
// bench.hpp (synthetic_case, run_sweep), dataset.hpp and protocol.hpp -- compile
// against it.  The clear and tlwe-oracle kinds keep the reference's semantics (same
// gate linear forms, gate_engine.hpp:196-269; same NoiseSampler draw order; same
// counting, :31-77; same exceptions, :304-320).
//
// The tfhe-b200 kind is the production backend the reference names at its plug-in
// point (gate_engine.hpp:113-123): real TFHE gate bootstrapping on the GPU through the
// C ABI of include/locpir_b200.h.  Gates are RECORDED, not executed: every hom_* call
// appends one op to the engine's pending program and returns a handle (a device pool
// slot).  The program is flushed -- planned into depth levels and run as batched
// blind-rotation / key-switch kernels (locpir_b200_run) -- when a result is needed on
// the host: decrypt(), CipherBit::sample() or refresh().  Encryption and decryption stay
// client-side (host), exactly as the oracle engine does them.
//
// Differences a caller can observe, all deliberate:
//  * check_pair accepts, besides the engine's own bits, TLWE samples of the
//    tlwe-oracle kind (e.g. encrypt_word(w, sk, sampler), codec.hpp:111-119): they are
//    valid inputs under the same key and are uploaded on the next flush.
//  * fork() children share the recorder (one GPU context, guarded by a mutex): gates
//    on distinct bits may be recorded concurrently from forks, as circuits.hpp's
//    parallel_blocks workers do (gate_engine.hpp:128-129).
//  * A bootstrap is deterministic, so fork noise streams only affect encrypt().
//  * Pool slots are reference-counted: a slot is reused once no CipherBit refers to
//    it and the program that might still read it has run.
#pragma once

#include <algorithm>
#include <atomic>
#include <cassert>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <string_view>
#include <variant>
#include <vector>

#include "locpir/torus.hpp"
#include "locpir_b200.h"

namespace locpir {

enum class EngineKind : uint8_t { Clear = 0, TlweOracle = 1, TfheB200 = 2 };

inline const char* engine_kind_name(EngineKind k)
{
    switch (k) {
    case EngineKind::Clear:
        return "clear";
    case EngineKind::TlweOracle:
        return "tlwe-oracle";
    default:
        return "tfhe-b200";
    }
}

inline EngineKind parse_engine_kind(std::string_view s)
{
    for (EngineKind k : {EngineKind::Clear, EngineKind::TlweOracle, EngineKind::TfheB200})
        if (s == engine_kind_name(k))
            return k;
    // "tfhe" keeps throwing (test_gate_engine.cpp:154)
    throw std::invalid_argument("unknown engine \"" + std::string(s) +
                                "\" (expected clear or tlwe-oracle)");
}

// ---- gate accounting (gate_engine.hpp:31-77): NOT is free, MUX costs two units
struct GateCounterSnapshot {
    uint64_t and_gates = 0, or_gates = 0, xor_gates = 0, xnor_gates = 0, not_gates = 0,
             mux_gates = 0;

    uint64_t bootstrap_units() const
    {
        return and_gates + or_gates + xor_gates + xnor_gates + 2 * mux_gates;
    }

    std::map<std::string, uint64_t> as_map() const
    {
        std::map<std::string, uint64_t> m;
        m["and"] = and_gates;
        m["or"] = or_gates;
        m["xor"] = xor_gates;
        m["xnor"] = xnor_gates;
        m["not"] = not_gates;
        m["mux"] = mux_gates;
        m["bootstrap_units"] = bootstrap_units();
        return m;
    }
};

class GateCounter {
public:
    enum Kind { And, Or, Xor, Xnor, Not, Mux, Kinds };

    GateCounterSnapshot snapshot() const
    {
        GateCounterSnapshot s;
        s.and_gates = c_[And].load();
        s.or_gates = c_[Or].load();
        s.xor_gates = c_[Xor].load();
        s.xnor_gates = c_[Xnor].load();
        s.not_gates = c_[Not].load();
        s.mux_gates = c_[Mux].load();
        return s;
    }
    void reset()
    {
        for (auto& x : c_)
            x.store(0);
    }
    void count(Kind k) { c_[k].fetch_add(1, std::memory_order_relaxed); }
    void count_and() { count(And); }
    void count_or() { count(Or); }
    void count_xor() { count(Xor); }
    void count_xnor() { count(Xnor); }
    void count_not() { count(Not); }
    void count_mux() { count(Mux); }

private:
    std::atomic<uint64_t> c_[Kinds]{};
};

// ---- the B200 recorder ------------------------------------------------------
namespace b200 {

inline void check(int rc, const locpir_b200_ctx* ctx)
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

// One GPU context with its evaluation keys, the pending gate program and the slot
// allocator.  Shared by every copy and fork of a tfhe-b200 GateEngine and by every
// handle it issued.
class State {
public:
    State(const locpir_b200_params& p, const std::vector<uint8_t>& lwe_key, uint64_t key_seed,
          int device)
        : p_(p)
    {
        check(locpir_b200_ctx_create(&p_, device, nullptr, &ctx_), nullptr);
        std::vector<uint32_t> bk(locpir_b200_bk_words(&p_)), ksk(locpir_b200_ksk_words(&p_));
        check(locpir_b200_keygen_with_lwe_key(&p_, key_seed, lwe_key.data(), nullptr, bk.data(),
                                              ksk.data()),
              ctx_);
        check(locpir_b200_upload_keys(ctx_, bk.data(), ksk.data(), 0), ctx_);
    }
    ~State()
    {
        if (ctx_)
            locpir_b200_ctx_destroy(ctx_);
    }
    State(const State&) = delete;
    State& operator=(const State&) = delete;

    uint32_t n() const { return p_.n; }

    // new slot written by a recorded op
    uint32_t record(uint32_t kind, uint32_t a, uint32_t b, uint32_t c)
    {
        std::lock_guard<std::mutex> g(mu_);
        const uint32_t out = alloc_locked();
        ops_.push_back({kind, a, b, c, out});
        return out;
    }
    // new slot holding a host sample (uploaded on the next flush)
    uint32_t upload(const TlweSample& s)
    {
        if (s.mask.size() != p_.n)
            throw std::invalid_argument("sample/key dimension mismatch");
        std::lock_guard<std::mutex> g(mu_);
        const uint32_t slot = alloc_locked();
        Up u{slot, std::vector<uint32_t>(p_.n + 1)};
        for (uint32_t i = 0; i < p_.n; i++)
            u.words[i] = s.mask[i].raw;
        u.words[p_.n] = s.body.raw;
        ups_.push_back(std::move(u));
        return slot;
    }
    // the handle of `slot` is gone: reusable after the program that may read it ran
    void release(uint32_t slot)
    {
        std::lock_guard<std::mutex> g(mu_);
        deferred_.push_back(slot);
    }
    void flush()
    {
        std::lock_guard<std::mutex> g(mu_);
        flush_locked();
    }
    TlweSample read(uint32_t slot)
    {
        std::lock_guard<std::mutex> g(mu_);
        flush_locked();
        std::vector<uint32_t> w(p_.n + 1);
        check(locpir_b200_pool_d2h(ctx_, slot, 1, w.data()), ctx_);
        TlweSample s{std::vector<Torus32>(p_.n), Torus32{w[p_.n]}};
        for (uint32_t i = 0; i < p_.n; i++)
            s.mask[i] = Torus32{w[i]};
        return s;
    }

private:
    struct Up {
        uint32_t slot;
        std::vector<uint32_t> words;
    };

    uint32_t alloc_locked()
    {
        if (!free_.empty()) {
            const uint32_t s = free_.back();
            free_.pop_back();
            return s;
        }
        if (next_ == 0xFFFFFFFEu)
            throw std::runtime_error("device pool slot space exhausted");
        return next_++;
    }
    void flush_locked()
    {
        if (ops_.empty() && ups_.empty())
            return;
        check(locpir_b200_pool_reserve(ctx_, next_), ctx_);
        std::sort(ups_.begin(), ups_.end(), [](const Up& a, const Up& b) { return a.slot < b.slot; });
        for (size_t i = 0; i < ups_.size();) {  // one copy per run of consecutive slots
            size_t j = i + 1;
            while (j < ups_.size() && ups_[j].slot == ups_[j - 1].slot + 1)
                j++;
            std::vector<uint32_t> buf;
            buf.reserve((j - i) * (p_.n + 1));
            for (size_t k = i; k < j; k++)
                buf.insert(buf.end(), ups_[k].words.begin(), ups_[k].words.end());
            check(locpir_b200_pool_h2d(ctx_, ups_[i].slot, j - i, buf.data()), ctx_);
            i = j;
        }
        ups_.clear();
        if (!ops_.empty()) {
            check(locpir_b200_run(ctx_, ops_.data(), ops_.size()), ctx_);
            ops_.clear();
        }
        free_.insert(free_.end(), deferred_.begin(), deferred_.end());
        deferred_.clear();
    }

    locpir_b200_params p_{};
    locpir_b200_ctx* ctx_ = nullptr;
    std::mutex mu_;
    std::vector<locpir_b200_gate_op> ops_;
    std::vector<Up> ups_;
    std::vector<uint32_t> free_, deferred_;
    uint32_t next_ = 0;
};

// A device-resident bit: one pool slot, written once.
struct Node {
    Node(std::shared_ptr<State> st, uint32_t slot) : state(std::move(st)), slot(slot) {}
    ~Node() { state->release(slot); }
    Node(const Node&) = delete;
    Node& operator=(const Node&) = delete;

    const TlweSample& sample() const
    {
        std::call_once(once_, [&] { cached_ = state->read(slot); });
        return cached_;
    }

    std::shared_ptr<State> state;
    uint32_t slot;

private:
    mutable std::once_flag once_;
    mutable TlweSample cached_;
};

}  // namespace b200

// One encrypted bit: a plain bit (clear), a host TLWE sample (tlwe-oracle) or a handle
// to a device slot (tfhe-b200).
class CipherBit {
public:
    CipherBit() : v_(false) {}
    explicit CipherBit(bool b) : v_(b) {}
    explicit CipherBit(TlweSample s) : v_(std::move(s)) {}
    explicit CipherBit(std::shared_ptr<b200::Node> n) : v_(std::move(n)) {}

    EngineKind kind() const
    {
        return v_.index() == 0 ? EngineKind::Clear
               : v_.index() == 1 ? EngineKind::TlweOracle
                                 : EngineKind::TfheB200;
    }

    bool clear_bit() const
    {
        if (const bool* b = std::get_if<bool>(&v_))
            return *b;
        throw std::invalid_argument("cipher bit is not a clear-engine bit");
    }

    // tfhe-b200: runs the pending program if needed and reads the slot back once
    const TlweSample& sample() const
    {
        if (const TlweSample* s = std::get_if<TlweSample>(&v_))
            return *s;
        if (const auto* n = std::get_if<std::shared_ptr<b200::Node>>(&v_))
            return (*n)->sample();
        throw std::invalid_argument("cipher bit carries no TLWE sample");
    }

    const b200::Node* node() const
    {
        const auto* n = std::get_if<std::shared_ptr<b200::Node>>(&v_);
        return n ? n->get() : nullptr;
    }

private:
    std::variant<bool, TlweSample, std::shared_ptr<b200::Node>> v_;
};

// The reference's secret-key refresh stand-in (gate_engine.hpp:117-123): threshold the
// phase, re-encrypt fresh.  Used by the tlwe-oracle kind only.
inline TlweSample bootstrap_oracle(const TlweSample& c, const SecretKey& sk,
                                   NoiseSampler& sampler)
{
    const uint32_t p = phase(c, sk).raw;
    return encrypt_bit(p != 0 && p <= 0x80000000u, sk, sampler);
}

class GateEngine {
public:
    static GateEngine make_clear() { return GateEngine(EngineKind::Clear, nullptr, 0, nullptr); }

    static GateEngine make_tlwe_oracle(SecretKey sk, uint64_t seed)
    {
        sk.params.validate();
        return GateEngine(EngineKind::TlweOracle, std::make_shared<const SecretKey>(std::move(sk)),
                          seed, nullptr);
    }

    // tfhe-b200 on a BASELINE.json parameter set (security_bits 80 or 128): the LWE key
    // is the reference keygen(n, key_seed) (torus.hpp:146-154); TRLWE key, BK and KSK
    // derive from key_seed (locpir_b200_keygen); `seed` drives encrypt() as for the oracle.
    static GateEngine make_tfhe_b200(int security_bits, uint64_t key_seed, uint64_t seed = 0,
                                     int device = 0)
    {
        locpir_b200_params p{};
        b200::check(locpir_b200_params_default(security_bits, &p), nullptr);
        const TlweParams tp = TlweParams::custom(p.n, p.alpha_in);
        SecretKey sk = keygen(tp, key_seed);
        auto st = std::make_shared<b200::State>(p, sk.bits, key_seed, device);
        return GateEngine(EngineKind::TfheB200, std::make_shared<const SecretKey>(std::move(sk)),
                          seed, std::move(st));
    }

    // tfhe-b200 around a reference SecretKey (e.g. keygen(TlweParams::sec128(), s)): the
    // gadget / ring parameters of the nearest BASELINE set (128-bit for n >= 600, else
    // 80-bit), LWE noise sigma from the key's params; TRLWE key, BK and KSK from key_seed.
    static GateEngine make_tfhe_b200(SecretKey sk, uint64_t key_seed, uint64_t seed,
                                     int device = 0)
    {
        sk.params.validate();
        locpir_b200_params p{};
        b200::check(locpir_b200_params_default(sk.params.n >= 600 ? 128 : 80, &p), nullptr);
        p.n = sk.params.n;
        p.alpha_in = sk.params.sigma;
        auto st = std::make_shared<b200::State>(p, sk.bits, key_seed, device);
        return GateEngine(EngineKind::TfheB200, std::make_shared<const SecretKey>(std::move(sk)),
                          seed, std::move(st));
    }

    GateEngine fork(uint64_t lane) const
    {
        GateEngine child(*this);
        child.seed_ = mix(seed_, lane);
        child.sampler_ = NoiseSampler(child.seed_, sigma());
        return child;
    }

    uint64_t acquire_fork_block() const { return fork_blocks_->fetch_add(1); }

    EngineKind kind() const { return kind_; }

    const TlweParams& params() const
    {
        need_key();
        return key_->params;
    }
    const SecretKey& secret_key() const
    {
        need_key();
        return *key_;
    }

    GateCounter& counters() { return *counters_; }
    const GateCounter& counters() const { return *counters_; }

    // trivial (noiseless) bit, no gate
    CipherBit constant(bool b) const
    {
        switch (kind_) {
        case EngineKind::Clear:
            return CipherBit(b);
        case EngineKind::TlweOracle:
            return CipherBit(trivial_sample(encode_bit(b), key_->params));
        default:
            return handle(dev_->record(LOCPIR_B200_CONST, b ? 1u : 0u, LOCPIR_B200_NONE_SLOT,
                                       LOCPIR_B200_NONE_SLOT));
        }
    }

    CipherBit encrypt(bool b)
    {
        if (kind_ == EngineKind::Clear)
            return CipherBit(b);
        TlweSample s = encrypt_bit(b, *key_, sampler_);
        if (kind_ == EngineKind::TlweOracle)
            return CipherBit(std::move(s));
        return handle(dev_->upload(s));
    }

    bool decrypt(const CipherBit& c) const
    {
        if (c.kind() == EngineKind::Clear)
            return c.clear_bit();
        need_key();
        return decrypt_bit(c.sample(), *key_);
    }

    CipherBit hom_and(const CipherBit& a, const CipherBit& b) { return gate2(And, a, b); }
    CipherBit hom_or(const CipherBit& a, const CipherBit& b) { return gate2(Or, a, b); }
    CipherBit hom_xor(const CipherBit& a, const CipherBit& b) { return gate2(Xor, a, b); }
    CipherBit hom_xnor(const CipherBit& a, const CipherBit& b) { return gate2(Xnor, a, b); }

    CipherBit hom_not(const CipherBit& a) const
    {
        check_bit(a);
        counters_->count_not();
        switch (kind_) {
        case EngineKind::Clear:
            return CipherBit(!a.clear_bit());
        case EngineKind::TlweOracle:
            return CipherBit(neg_sample(a.sample()));
        default:
            return handle(dev_->record(LOCPIR_B200_NOT, slot_of(a), LOCPIR_B200_NONE_SLOT,
                                       LOCPIR_B200_NONE_SLOT));
        }
    }

    // sel ? a : b, two units (gate_engine.hpp:254-269).  tfhe-b200: TFHE bootsMUX, two
    // blind rotations without key switch, one key switch of their sum + 1/8.
    CipherBit hom_mux(const CipherBit& sel, const CipherBit& a, const CipherBit& b)
    {
        check_pair(sel, a);
        check_pair(sel, b);
        counters_->count_mux();
        switch (kind_) {
        case EngineKind::Clear:
            return CipherBit(sel.clear_bit() ? a.clear_bit() : b.clear_bit());
        case EngineKind::TlweOracle: {
            const TlweSample off = trivial_sample({0xE0000000u}, key_->params);
            TlweSample u = refresh(add_samples(add_samples(off, sel.sample()), a.sample()));
            TlweSample v = refresh(add_samples(add_samples(off, neg_sample(sel.sample())),
                                               b.sample()));
            return CipherBit(refresh_gate(
                add_samples(add_samples(u, v), trivial_sample({0x20000000u}, key_->params))));
        }
        default:
            return handle(dev_->record(LOCPIR_B200_MUX, slot_of(sel), slot_of(a), slot_of(b)));
        }
    }

    // one bootstrap of c, counted nowhere (noise experiments).  tfhe-b200: OR(c, Enc(0)),
    // whose linear form 1/8 + c - 1/8 is c itself, bootstrapped on the GPU.
    TlweSample refresh(const TlweSample& c)
    {
        need_key();
        if (kind_ == EngineKind::TlweOracle)
            return bootstrap_oracle(c, *key_, sampler_);
        const uint32_t zero = dev_->record(LOCPIR_B200_CONST, 0u, LOCPIR_B200_NONE_SLOT,
                                           LOCPIR_B200_NONE_SLOT);
        const uint32_t in = dev_->upload(c);
        CipherBit z = handle(zero), x = handle(in);
        return handle(dev_->record(LOCPIR_B200_OR, in, zero, LOCPIR_B200_NONE_SLOT)).sample();
    }

    // tfhe-b200: run every recorded gate now (decrypt / sample() do this on demand)
    void flush()
    {
        if (dev_)
            dev_->flush();
    }

private:
    enum Gate2 { And, Or, Xor, Xnor };

    GateEngine(EngineKind kind, std::shared_ptr<const SecretKey> key, uint64_t seed,
               std::shared_ptr<b200::State> dev)
        : kind_(kind),
          key_(std::move(key)),
          counters_(std::make_shared<GateCounter>()),
          fork_blocks_(std::make_shared<std::atomic<uint64_t>>(0)),
          seed_(seed),
          sampler_(seed, key_ ? key_->params.sigma : 0.0),
          dev_(std::move(dev))
    {
    }

    // the reference's fork lane mixer (splitmix64 finaliser, gate_engine.hpp:296-302)
    static uint64_t mix(uint64_t seed, uint64_t lane)
    {
        uint64_t x = seed + 0x9e3779b97f4a7c15ull * (lane + 1);
        x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
        x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
        return x ^ (x >> 31);
    }
    double sigma() const { return key_ ? key_->params.sigma : 0.0; }

    void need_key() const
    {
        if (!key_)
            throw std::logic_error("operation requires the tlwe-oracle engine");
    }
    bool accepts(const CipherBit& c) const
    {
        if (c.kind() == kind_)
            return kind_ != EngineKind::TfheB200 || c.node()->state == dev_;
        return kind_ == EngineKind::TfheB200 && c.kind() == EngineKind::TlweOracle;
    }
    void check_bit(const CipherBit& c) const
    {
        if (!accepts(c))
            throw std::invalid_argument("cipher bit belongs to a different engine");
    }
    void check_pair(const CipherBit& a, const CipherBit& b) const
    {
        check_bit(a);
        check_bit(b);
    }

    CipherBit handle(uint32_t slot) const
    {
        return CipherBit(std::make_shared<b200::Node>(dev_, slot));
    }
    // operand slot; host samples of the oracle kind are uploaded with the program
    uint32_t slot_of(const CipherBit& c) const
    {
        if (const b200::Node* n = c.node())
            return n->slot;
        const uint32_t s = dev_->upload(c.sample());
        dev_->release(s);  // no handle: reusable once this program has run
        return s;
    }

    // reference linear forms (gate_engine.hpp:196-240): offset + k (a + b)
    CipherBit gate2(Gate2 g, const CipherBit& a, const CipherBit& b)
    {
        check_pair(a, b);
        static const GateCounter::Kind ck[] = {GateCounter::And, GateCounter::Or,
                                               GateCounter::Xor, GateCounter::Xnor};
        counters_->count(ck[g]);
        if (kind_ == EngineKind::Clear) {
            const bool x = a.clear_bit(), y = b.clear_bit();
            return CipherBit(g == And ? (x && y) : g == Or ? (x || y) : g == Xor ? x != y : x == y);
        }
        if (kind_ == EngineKind::TlweOracle) {
            static const uint32_t off[] = {0xE0000000u, 0x20000000u, 0x40000000u, 0xC0000000u};
            static const int32_t k[] = {1, 1, 2, -2};
            const TlweSample sa = k[g] == 1 ? a.sample() : scale_sample(k[g], a.sample());
            const TlweSample sb = k[g] == 1 ? b.sample() : scale_sample(k[g], b.sample());
            return CipherBit(refresh_gate(
                add_samples(add_samples(trivial_sample({off[g]}, key_->params), sa), sb)));
        }
        static const uint32_t kind[] = {LOCPIR_B200_AND, LOCPIR_B200_OR, LOCPIR_B200_XOR,
                                        LOCPIR_B200_XNOR};
        return handle(dev_->record(kind[g], slot_of(a), slot_of(b), LOCPIR_B200_NONE_SLOT));
    }

    TlweSample refresh_gate(const TlweSample& combo)
    {
        // a valid gate input keeps the combined phase clear of the decision boundary
        assert(std::abs(torus_to_double(phase(combo, *key_))) > 1.0 / 64);
        return bootstrap_oracle(combo, *key_, sampler_);
    }

    EngineKind kind_;
    std::shared_ptr<const SecretKey> key_;
    std::shared_ptr<GateCounter> counters_;
    std::shared_ptr<std::atomic<uint64_t>> fork_blocks_;
    uint64_t seed_;
    NoiseSampler sampler_;
    std::shared_ptr<b200::State> dev_;
};

}  // namespace locpir
