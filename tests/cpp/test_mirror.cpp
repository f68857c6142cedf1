// test_mirror.cpp -- the reference's own engine/circuit tests, restated against the
// C++ mirror (paper_2407_19871_b200/host/locpir_b200.hpp) of the B200 engine.
// Mirrors test_gate_engine.cpp:17-97 and test_circuits.cpp:26-213 (Catch2 is not in
// this image; a tiny CHECK macro stands in).  Driven by tests/test_cpp_mirror.py.
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <functional>
#include <stdexcept>

#include "../../paper_2407_19871_b200/host/locpir_b200.hpp"

using namespace locpir_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(x)                                                                   \
    do {                                                                           \
        g_checks++;                                                                \
        if (!(x)) {                                                                \
            g_fail++;                                                              \
            std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #x); \
        }                                                                          \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                  \
    do {                                          \
        bool thrown_ = false;                     \
        try {                                     \
            (void)(expr);                         \
        } catch (const T&) {                      \
            thrown_ = true;                       \
        }                                         \
        CHECK(thrown_);                           \
    } while (0)

static CipherWord enc_int(int64_t v, int l, GateEngine& e)
{
    std::vector<uint8_t> bits(l);
    const uint64_t u = static_cast<uint64_t>(v);
    for (int i = 0; i < l; i++)
        bits[i] = (u >> i) & 1;
    return {e.encrypt_many(bits)};
}

static CipherWord const_int(int64_t v, int l, GateEngine& e)
{
    CipherWord w;
    BatchScope s(e);
    const uint64_t u = static_cast<uint64_t>(v);
    for (int i = 0; i < l; i++)
        w.bits.push_back(e.constant((u >> i) & 1));
    return w;
}

static uint64_t dec_service(const ServiceCiphertext& s, GateEngine& e)
{
    uint64_t v = 0;
    for (size_t j = 0; j < s.bits.size(); j++)
        if (e.decrypt(s.bits[j]))
            v |= 1ull << j;
    return v;
}

int main()
{
    const ClientKeys keys(Params::tfhe80(), 42);
    GateEngine eng = GateEngine::make_b200(keys, 43);

    // test_gate_engine.cpp:17-38 truth tables
    for (int a = 0; a <= 1; a++)
        for (int b = 0; b <= 1; b++) {
            const CipherBit ca = eng.encrypt(a), cb = eng.encrypt(b);
            CHECK(eng.decrypt(eng.hom_and(ca, cb)) == (a && b));
            CHECK(eng.decrypt(eng.hom_or(ca, cb)) == (a || b));
            CHECK(eng.decrypt(eng.hom_xor(ca, cb)) == (a != b));
            CHECK(eng.decrypt(eng.hom_xnor(ca, cb)) == (a == b));
            CHECK(eng.decrypt(eng.hom_nand(ca, cb)) == !(a && b));
            CHECK(eng.decrypt(eng.hom_not(ca)) == !a);
            for (int s = 0; s <= 1; s++) {
                const CipherBit cs = eng.encrypt(s);
                CHECK(eng.decrypt(eng.hom_mux(cs, ca, cb)) == (s ? a : b));
            }
        }

    // test_gate_engine.cpp:40-69 counters
    {
        eng.reset_counters();
        const CipherBit a = eng.encrypt(true), b = eng.encrypt(false);
        (void)eng.hom_and(a, b);
        (void)eng.hom_or(a, b);
        (void)eng.hom_or(a, b);
        (void)eng.hom_xor(a, b);
        (void)eng.hom_xnor(a, b);
        (void)eng.hom_not(a);
        (void)eng.hom_mux(a, a, b);
        (void)eng.constant(true);
        const GateCounterSnapshot s = eng.counters();
        CHECK(s.and_gates == 1 && s.or_gates == 2 && s.xor_gates == 1 && s.xnor_gates == 1);
        CHECK(s.not_gates == 1 && s.mux_gates == 1);
        CHECK(s.bootstrap_units() == 1 + 2 + 1 + 1 + 2 * 1);
        CHECK(s.as_map().at("bootstrap_units") == s.bootstrap_units());
    }

    // test_gate_engine.cpp:140-155 errors
    {
        GateEngine other = GateEngine::make_b200(keys, 44);
        const CipherBit mine = eng.encrypt(true);
        CHECK_THROWS_AS(other.hom_and(mine, mine), std::invalid_argument);
        CHECK(parse_engine_kind("tfhe-b200") == EngineKind::TfheB200);
        CHECK_THROWS_AS(parse_engine_kind("tfhe"), std::invalid_argument);
    }

    // test_circuits.cpp:26-40 comparator vs signed order at l = 6 (batched per pair set)
    {
        const int l = 6;
        const int64_t vals[] = {-32, -17, -1, 0, 1, 17, 31};
        std::vector<std::tuple<int64_t, int64_t, CipherBit, CipherBit>> res;
        std::vector<std::tuple<int64_t, int64_t, CipherBit>> majres;
        {
            std::vector<std::pair<CipherWord, CipherWord>> words;
            for (int64_t a : vals)
                for (int64_t b : vals)
                    words.push_back({enc_int(a, l, eng), enc_int(b, l, eng)});
            BatchScope scope(eng);
            size_t k = 0;
            for (int64_t a : vals)
                for (int64_t b : vals) {
                    const auto& w = words[k++];
                    res.emplace_back(a, b, hom_less(w.first, w.second, eng),
                                     hom_less_equal(w.first, w.second, eng));
                    majres.emplace_back(a, b, hom_less_maj(w.first, w.second, eng));
                }
        }
        for (auto& [a, b, lt, le] : res) {
            CHECK(eng.decrypt(lt) == (a < b));
            CHECK(eng.decrypt(le) == (a <= b));
        }
        for (auto& [a, b, lt] : majres)  // flagged majority-borrow comparator
            CHECK(eng.decrypt(lt) == (a < b));
    }

    // test_circuits.cpp:150-213 loc_pir retrieval, half-open edges, counts
    {
        const int l = 6;
        auto regions_for = [&]() {
            std::vector<EncodedRegion> r(3);
            BatchScope s(eng);
            const int64_t spec[3][4] = {{0, 8, 0, 8}, {8, 16, 0, 8}, {-16, -4, -12, -4}};
            const uint64_t svc[3] = {5, 3, 7};
            for (int i = 0; i < 3; i++) {
                r[i].x1 = const_int(spec[i][0], l, eng);
                r[i].x2 = const_int(spec[i][1], l, eng);
                r[i].y1 = const_int(spec[i][2], l, eng);
                r[i].y2 = const_int(spec[i][3], l, eng);
                for (int j = 0; j < 3; j++)
                    r[i].service.bits.push_back(eng.constant((svc[i] >> j) & 1));
                r[i].region_id = i;
            }
            return r;
        };
        const auto regions = regions_for();
        const std::pair<std::pair<int64_t, int64_t>, uint64_t> cases[] = {
            {{5, 2}, 5}, {{9, 1}, 3}, {{-10, -6}, 7}, {{28, 28}, 0},
            {{0, 0}, 5}, {{8, 0}, 3}, {{16, 0}, 0},   {{5, 8}, 0}};
        eng.reset_counters();
        for (bool tree : {false, true})
            for (const auto& [pt, want] : cases) {
                const CipherWord x = enc_int(pt.first, l, eng), y = enc_int(pt.second, l, eng);
                CHECK(dec_service(loc_pir(x, y, regions, eng, tree), eng) == want);
            }
        const GateCounterSnapshot s = eng.counters();
        const uint64_t q = 16, N = 3, m = 3;
        CHECK(s.xnor_gates == q * N * 4 * l && s.mux_gates == q * N * 4 * l);
        CHECK(s.and_gates == q * N * (3 + m) && s.xor_gates == q * N * m);
        CHECK(s.bootstrap_units() == q * N * (12 * l + 2 * m + 3));
        eng.reset_counters();
        for (const auto& [pt, want] : cases) {  // flagged majority comparators: same answers
            const CipherWord x = enc_int(pt.first, l, eng), y = enc_int(pt.second, l, eng);
            CHECK(dec_service(loc_pir(x, y, regions, eng, true, Comparator::Majority), eng) == want);
        }
        CHECK(eng.counters().bootstrap_units() == 8 * N * (4 * l + 2 * m + 3));
        // the reference's argument checks (circuits.hpp:283-292)
        {
            const CipherWord x = enc_int(1, l, eng), y = enc_int(2, l, eng);
            CipherWord y13 = y;
            y13.int_bits = 9;
            y13.frac_bits = 4;
            CHECK_THROWS_AS(loc_pir(x, y13, regions, eng), std::invalid_argument);
            auto bad = regions;
            bad[1].service.bits.pop_back();
            CHECK_THROWS_AS(loc_pir(x, y, bad, eng), std::invalid_argument);
            bad = regions;
            bad[0].x2.bits.pop_back();
            CHECK_THROWS_AS(loc_pir(x, y, bad, eng), std::invalid_argument);
        }
    }

    // majority gate truth table (one bootstrap of a + b + c)
    for (int a = 0; a <= 1; a++)
        for (int b = 0; b <= 1; b++)
            for (int c = 0; c <= 1; c++) {
                const CipherBit ca = eng.encrypt(a), cb = eng.encrypt(b), cc = eng.encrypt(c);
                CHECK(eng.decrypt(eng.hom_maj(ca, cb, cc)) == (a + b + c >= 2));
            }

    // cross-session batcher through wire payloads (protocol.hpp:185-227)
    {
        const uint32_t l = 16, m = 4;
        const std::vector<int64_t> boxes = {0, 100, 0, 100, -50, 20, -30, 10, 200, 300, -5, 5};
        const std::vector<uint64_t> services = {9, 6, 13};
        // engine values from before the server exists must survive it (the
        // server owns a disjoint pool tail, the engine's slots stay below it)
        const CipherBit before1 = eng.hom_xor(eng.encrypt(1), eng.encrypt(0));
        const CipherBit before0 = eng.hom_and(eng.encrypt(1), eng.encrypt(0));
        BatchingServer srv(eng, boxes, services, l, m, 2);
        const size_t S = keys.params.sample_words();
        auto sheet = [&](uint64_t seed) {  // Enc(-1/8) + 1/8 = Enc(0) per sample
            auto cts = keys.encrypt(std::vector<uint8_t>(services.size() * m, 0), seed);
            for (size_t i = 0; i < services.size() * m; i++)
                cts[i * S + S - 1] += 0x20000000u;
            std::vector<uint8_t> b(cts.size() * 4);
            std::memcpy(b.data(), cts.data(), b.size());
            return b;
        };
        const uint32_t s0 = srv.open_session(sheet(501)), s1 = srv.open_session(sheet(502));
        auto query = [&](int64_t gx, int64_t gy, uint64_t seed) {
            std::vector<uint8_t> out;
            for (int64_t g : {gx, gy}) {
                std::vector<uint8_t> bits(l);
                for (uint32_t i = 0; i < l; i++)
                    bits[i] = ((uint64_t)g >> i) & 1;
                const auto cts = keys.encrypt(bits, seed++);
                out.push_back((uint8_t)l);
                const uint8_t* p = reinterpret_cast<const uint8_t*>(cts.data());
                out.insert(out.end(), p, p + cts.size() * 4);
            }
            return out;
        };
        const std::pair<std::pair<int64_t, int64_t>, uint64_t> qs[] = {
            {{50, 50}, 9}, {{0, -30}, 6}, {{250, 0}, 13}, {{-60, 0}, 0}, {{19, 9}, 6 ^ 9}};
        std::vector<uint64_t> tickets;
        uint64_t seed = 600;
        for (size_t i = 0; i < 5; i++, seed += 2)
            tickets.push_back(srv.submit(i % 2 ? s1 : s0, query(qs[i].first.first, qs[i].first.second, seed)));
        CHECK(srv.pending() == 5 && srv.flush() == 5);
        for (size_t i = 0; i < 5; i++) {
            const auto resp = srv.take_response(tickets[i]);
            std::vector<uint32_t> w(resp.size() / 4);
            std::memcpy(w.data(), resp.data(), resp.size());
            const auto bits = keys.decrypt(w);
            uint64_t v = 0;
            for (uint32_t j = 0; j < m; j++)
                v |= (uint64_t)bits[j] << j;
            CHECK(v == qs[i].second);
        }
        CHECK_THROWS_AS(srv.submit(7, query(1, 1, 9)), std::logic_error);
        // the engine keeps working next to the server, and its old values are intact
        CHECK(eng.decrypt(before1) == 1 && eng.decrypt(before0) == 0);
        CHECK(eng.decrypt(eng.hom_or(before1, before0)) == 1);
        // a raw ABI call into the server's slots is refused instead of corrupting them
        {
            const uint64_t tail = eng.reserve_server_tail();
            std::vector<uint32_t> row(keys.params.sample_words(), 0);
            CHECK(locpir_b200_pool_h2d(eng.native(), tail, 1, row.data()) == LOCPIR_B200_EINVAL);
        }
    }

    // slot arena: reset_slots() recycles the pool; bits from before a reset are rejected
    {
        const CipherBit old = eng.encrypt(1);
        const uint64_t used = eng.slots_in_use();
        eng.reset_slots();
        CHECK(eng.slots_in_use() == 0 && used > 0);
        CHECK_THROWS_AS(eng.decrypt(old), std::invalid_argument);
        CHECK(eng.decrypt(eng.hom_nand(eng.encrypt(1), eng.encrypt(1))) == 0);
    }

    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
