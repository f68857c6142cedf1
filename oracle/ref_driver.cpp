// ref_driver.cpp -- runs the UNMODIFIED reference headers (compiled read-only from
// /root/reference/proj/include, see oracle/Makefile) and prints golden vectors as
// JSON.  Test infrastructure only: tests/golden/make_golden.py runs it and commits
// the output as tests/golden/ref_vectors.json, which pins oracle/tfhe_oracle.c.
//
// Also provides the "stand-in" timing mode used by bench.py to report the
// reference's own refresh-oracle gate rate (gate_engine.hpp:117-123), labelled
// "functional stand-in, no bootstrapping".
#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "locpir/locpir.hpp"

using namespace locpir;

static void put_words(const char* key, const std::vector<uint32_t>& w, bool comma = true)
{
    std::printf("\"%s\": [", key);
    for (size_t i = 0; i < w.size(); i++)
        std::printf("%s%u", i ? "," : "", w[i]);
    std::printf("]%s\n", comma ? "," : "");
}

static std::vector<uint32_t> sample_words(const TlweSample& s)
{
    std::vector<uint32_t> w;
    for (auto t : s.mask)
        w.push_back(t.raw);
    w.push_back(s.body.raw);
    return w;
}

static int golden()
{
    std::printf("{\n");
    // keygen (torus.hpp:146-154)
    for (auto [name, p, seed] : {std::tuple{"keygen_sec80_seed11", TlweParams::sec80(), 11ull},
                                 std::tuple{"keygen_sec128_seed12", TlweParams::sec128(), 12ull},
                                 std::tuple{"keygen_n630_seed7", TlweParams::custom(630, std::exp2(-15)), 7ull}}) {
        SecretKey sk = keygen(p, seed);
        std::vector<uint32_t> bits(sk.bits.begin(), sk.bits.end());
        put_words(name, bits);
    }
    // raw sampler streams (torus.hpp:119-138)
    {
        NoiseSampler s(13, TlweParams::sec80().sigma);
        std::vector<uint32_t> g, u;
        for (int i = 0; i < 64; i++) {
            g.push_back(s.gaussian().raw);
            u.push_back(s.uniform().raw);
        }
        put_words("sampler13_sec80_gauss", g);
        put_words("sampler13_sec80_unif", u);
        NoiseSampler s2(99, std::exp2(-15));
        std::vector<uint32_t> g2;
        for (int i = 0; i < 256; i++)
            g2.push_back(s2.gaussian().raw);
        put_words("sampler99_a15_gauss", g2);
        NoiseSampler s3(5, std::exp2(-25));
        std::vector<uint32_t> g3;
        for (int i = 0; i < 256; i++)
            g3.push_back(s3.gaussian().raw);
        put_words("sampler5_a25_gauss", g3);
    }
    // encryptions (torus.hpp:161-175)
    {
        const TlweParams p = TlweParams::sec128();
        SecretKey sk = keygen(p, 12);
        NoiseSampler s(14, p.sigma);
        put_words("enc_sec128_k12_s14_bit1", sample_words(encrypt_bit(true, sk, s)));
        put_words("enc_sec128_k12_s14_bit0", sample_words(encrypt_bit(false, sk, s)));
        put_words("enc_sec128_k12_s14_mu0", sample_words(encrypt_torus({0}, sk, s)));
        TlweSample a = encrypt_bit(true, sk, s);
        put_words("phase_of_next", {phase(a, sk).raw});
        put_words("standin_refresh_of_next", sample_words(bootstrap_oracle(a, sk, s)));
    }
    {
        const TlweParams p = TlweParams::custom(630, std::exp2(-15));
        SecretKey sk = keygen(p, 7);
        NoiseSampler s(8, p.sigma);
        std::vector<uint32_t> all;
        for (int i = 0; i < 4; i++) {
            auto w = sample_words(encrypt_bit(i & 1, sk, s));
            all.insert(all.end(), w.begin(), w.end());
        }
        put_words("enc_n630_a15_k7_s8_four", all);
    }
    // oracle-engine gate outputs (gate_engine.hpp:196-269); deterministic per seed
    {
        GateEngine eng = GateEngine::make_tlwe_oracle(keygen(TlweParams::sec80(), 42), 43);
        std::vector<uint32_t> table;
        for (int a = 0; a <= 1; a++)
            for (int b = 0; b <= 1; b++) {
                CipherBit ca = eng.encrypt(a), cb = eng.encrypt(b);
                table.push_back(eng.decrypt(eng.hom_and(ca, cb)));
                table.push_back(eng.decrypt(eng.hom_or(ca, cb)));
                table.push_back(eng.decrypt(eng.hom_xor(ca, cb)));
                table.push_back(eng.decrypt(eng.hom_xnor(ca, cb)));
                table.push_back(eng.decrypt(eng.hom_not(ca)));
                for (int sl = 0; sl <= 1; sl++) {
                    CipherBit cs = eng.encrypt(sl);
                    table.push_back(eng.decrypt(eng.hom_mux(cs, ca, cb)));
                }
            }
        put_words("truth_table_and_or_xor_xnor_not_mux0_mux1", table);
        auto s = eng.counters().snapshot();
        put_words("truth_table_counters", {(uint32_t)s.and_gates, (uint32_t)s.or_gates,
                                           (uint32_t)s.xor_gates, (uint32_t)s.xnor_gates,
                                           (uint32_t)s.not_gates, (uint32_t)s.mux_gates,
                                           (uint32_t)s.bootstrap_units()});
    }
    // comparator (circuits.hpp:191-216) under the clear engine, l = 6 signed grid
    {
        GateEngine eng = GateEngine::make_clear();
        const FixedPointFormat fmt{4, 2};
        std::vector<uint32_t> lt, le;
        for (int64_t a = -32; a < 32; a += 3)
            for (int64_t b = -32; b < 32; b += 5) {
                CipherWord ca = encrypt_word(PlainWord::from_integer(a, fmt), eng);
                CipherWord cb = encrypt_word(PlainWord::from_integer(b, fmt), eng);
                lt.push_back(eng.decrypt(hom_less(ca, cb, eng)));
                le.push_back(eng.decrypt(hom_less_equal(ca, cb, eng)));
            }
        put_words("cmp_l6_lt_a_m32_s3_b_m32_s5", lt);
        put_words("cmp_l6_le_a_m32_s3_b_m32_s5", le);
    }
    // loc_pir synthetic sweep (bench.hpp:345-384) under the clear engine
    {
        std::vector<uint32_t> rows;
        for (uint32_t N : {1u, 3u, 9u, 16u})
            for (uint8_t l : {6, 13, 16})
                for (uint32_t m : {3u, 8u, 9u}) {
                    if ((int64_t)N * 4 >= (1ll << (l - 1)))
                        continue;
                    GateEngine eng = GateEngine::make_clear();
                    auto c = detail::synthetic_case(N, l, m, eng, nullptr, nullptr);
                    eng.counters().reset();
                    auto out = loc_pir(c.x, c.y, c.regions, eng, 1);
                    auto s = eng.counters().snapshot();
                    rows.insert(rows.end(),
                                {N, l, m, (uint32_t)decrypt_service(out, eng), (uint32_t)c.expected,
                                 (uint32_t)s.bootstrap_units(), (uint32_t)s.xnor_gates,
                                 (uint32_t)s.mux_gates, (uint32_t)s.and_gates, (uint32_t)s.xor_gates,
                                 (uint32_t)s.not_gates,
                                 (uint32_t)predict_gate_units(N, l, m)});
                }
        put_words("locpir_synthetic_N_l_m_got_expected_units_xnor_mux_and_xor_not_pred", rows);
    }
    // the 9-city KDCA table end to end (acceptance.cpp:180-237), clear engine: grid-encoded
    // boxes (dataset.hpp:232-259), services, interior query points + one outside point,
    // and the reference's own retrieved values
    {
        const FixedPointFormat fmt{9, 7};
        auto [records, dataset] = load_dataset("/root/reference/proj/data/kdca_2021-10-26.csv", fmt);
        GateEngine eng = GateEngine::make_clear();
        std::vector<uint64_t> services;
        std::vector<uint32_t> boxes, svc, queries, expected;
        for (const RegionRecord& r : records) {
            services.push_back(r.service);
            for (double v : {r.lat1, r.lat2, r.lon1, r.lon2})
                boxes.push_back((uint32_t)(int32_t)scale_to_grid(v, fmt));
            svc.push_back((uint32_t)r.service);
        }
        auto regions = encode_regions(records, fmt, eng,
                                      trivial_services(services, dataset.service_bits, eng));
        std::vector<std::pair<double, double>> pts;
        for (const RegionRecord& r : records)
            pts.push_back({(r.lat1 + r.lat2) / 2, (r.lon1 + r.lon2) / 2});
        pts.push_back({33.0, 127.0});
        for (auto [lat, lon] : pts) {
            const PlainWord px = encode_fixed(lat, fmt), py = encode_fixed(lon, fmt);
            queries.push_back((uint32_t)(int32_t)px.signed_value());
            queries.push_back((uint32_t)(int32_t)py.signed_value());
            auto out = loc_pir(constant_word(px, eng), constant_word(py, eng), regions, eng, 1);
            expected.push_back((uint32_t)decrypt_service(out, eng));
        }
        put_words("city_boxes_grid_x1_x2_y1_y2_int32", boxes);
        put_words("city_services", svc);
        put_words("city_service_bits", {dataset.service_bits});
        put_words("city_queries_grid_xy_int32", queries);
        put_words("city_expected", expected);
    }
    // wire payloads: QUERY = two framed words (codec.hpp:172-193,
    // protocol.hpp:185-193), ZEROSHEET = N*m raw zero samples (circuits.hpp:46-54, :83-89),
    // services preprocessed with the sheet (circuits.hpp:118-146), RESPONSE = m raw samples
    // (protocol.hpp:212-227).  Digests: FNV-1a 64 over the bytes, as (lo, hi) u32.
    {
        auto fnv = [](const std::vector<uint8_t>& b) {
            uint64_t h = 1469598103934665603ull;
            for (uint8_t c : b) {
                h ^= c;
                h *= 1099511628211ull;
            }
            return std::vector<uint32_t>{(uint32_t)h, (uint32_t)(h >> 32)};
        };
        const TlweParams p = TlweParams::sec128();
        SecretKey sk = keygen(p, 12);
        const FixedPointFormat fmt{9, 7};
        NoiseSampler s(17, p.sigma);
        const GeoCoordinate where(37.5665, 126.978);
        auto q = query_payload(where, fmt, sk, s);
        put_words("wire_query_len_lat_lon_grid",
                  {(uint32_t)q.size(), (uint32_t)(int32_t)scale_to_grid(where.lat, fmt),
                   (uint32_t)(int32_t)scale_to_grid(where.lon, fmt)});
        put_words("wire_query_fnv1a64", fnv(q));
        NoiseSampler s2(18, p.sigma);
        auto zs = zero_sheet_payload(sk, 3, 4, s2);
        put_words("wire_zerosheet_len", {(uint32_t)zs.size()});
        put_words("wire_zerosheet_fnv1a64", fnv(zs));
        auto sheet = ZeroSampleSheet::from_payload(zs, p, 3, 4);
        auto svc = preprocess_services({5, 9, 14}, sheet, 4);
        ByteWriter w;
        for (const auto& sc : svc)
            for (const auto& bit : sc.bits)
                write_sample(w, bit.sample());
        auto pre = w.take();
        put_words("wire_services_5_9_14_fnv1a64", fnv(pre));
        std::vector<uint8_t> resp(pre.begin() + 4 * sample_byte_size(p),
                                  pre.begin() + 8 * sample_byte_size(p));
        put_words("wire_response_region1_value", {(uint32_t)decrypt_response(resp, sk, 4)});
    }
    // sizes (acceptance.cpp:38-101)
    {
        put_words("sample_bytes_sec80_sec128",
                  {(uint32_t)sample_byte_size(TlweParams::sec80()),
                   (uint32_t)sample_byte_size(TlweParams::sec128())},
                  false);
    }
    std::printf("}\n");
    return 0;
}

// Times the reference refresh-oracle gates (NOT(AND)) on all host threads using the
// reference partitioner parallel_blocks (parallel.hpp:15-52).
static int standin(uint64_t gates, unsigned threads)
{
    const TlweParams p = TlweParams::sec128();
    GateEngine eng = GateEngine::make_tlwe_oracle(keygen(p, 1), 2);
    std::vector<CipherBit> a, b;
    for (uint64_t i = 0; i < gates; i++) {
        a.push_back(eng.encrypt(i & 1));
        b.push_back(eng.encrypt((i >> 1) & 1));
    }
    std::vector<CipherBit> out(gates);
    const uint64_t block = eng.acquire_fork_block();
    auto t0 = std::chrono::steady_clock::now();
    parallel_blocks(gates, threads, [&](unsigned w, size_t lo, size_t hi) {
        GateEngine local = eng.fork((block << 16) | w);
        for (size_t i = lo; i < hi; i++)
            out[i] = local.hom_not(local.hom_and(a[i], b[i]));
    });
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    uint64_t bad = 0;
    for (uint64_t i = 0; i < gates; i++)
        bad += eng.decrypt(out[i]) != !((i & 1) && ((i >> 1) & 1));
    std::printf("{\"gates\": %llu, \"threads\": %u, \"seconds\": %.6f, \"gates_per_s\": %.3f, \"wrong\": %llu}\n",
                (unsigned long long)gates, threads, secs, gates / secs, (unsigned long long)bad);
    return bad ? 1 : 0;
}

// Times the reference loc_pir (circuits.hpp:276-324) under the refresh-oracle engine on
// the reference's synthetic case (bench.hpp:150-189) with `threads` region workers.
static int standin_locpir(uint32_t N, uint8_t l, uint32_t m, int sec, uint32_t queries,
                          unsigned threads)
{
    const TlweParams p = sec == 80 ? TlweParams::sec80() : TlweParams::sec128();
    GateEngine eng = GateEngine::make_tlwe_oracle(keygen(p, 1), 2);
    auto c = detail::synthetic_case(N, l, m, eng, nullptr, nullptr);
    uint64_t wrong = 0;
    auto t0 = std::chrono::steady_clock::now();
    for (uint32_t q = 0; q < queries; q++) {
        auto out = loc_pir(c.x, c.y, c.regions, eng, threads);
        wrong += decrypt_service(out, eng) != c.expected;
    }
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("{\"queries\": %u, \"threads\": %u, \"seconds\": %.6f, \"queries_per_s\": %.6f, "
                "\"wrong\": %llu}\n",
                queries, threads, secs, queries / secs, (unsigned long long)wrong);
    return wrong ? 1 : 0;
}

int main(int argc, char** argv)
{
    if (argc >= 8 && std::strcmp(argv[1], "standin_locpir") == 0)
        return standin_locpir((uint32_t)std::strtoul(argv[2], nullptr, 10),
                              (uint8_t)std::strtoul(argv[3], nullptr, 10),
                              (uint32_t)std::strtoul(argv[4], nullptr, 10), std::atoi(argv[5]),
                              (uint32_t)std::strtoul(argv[6], nullptr, 10),
                              (unsigned)std::strtoul(argv[7], nullptr, 10));
    if (argc >= 2 && std::strcmp(argv[1], "golden") == 0)
        return golden();
    if (argc >= 2 && std::strcmp(argv[1], "standin") == 0) {
        uint64_t gates = argc >= 3 ? std::strtoull(argv[2], nullptr, 10) : 65536;
        unsigned threads = argc >= 4 ? (unsigned)std::strtoul(argv[3], nullptr, 10)
                                     : std::max(1u, std::thread::hardware_concurrency());
        return standin(gates, threads);
    }
    std::fprintf(stderr, "usage: ref_driver golden | standin [gates] [threads] | "
                         "standin_locpir N l m sec queries threads\n");
    return 2;
}
