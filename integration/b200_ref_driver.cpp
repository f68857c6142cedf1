// b200_ref_driver -- the reference's UNMODIFIED circuits (circuits.hpp: hom_less,
// mask_service, xor_sum_services, loc_pir; codec.hpp: constant_word, encrypt_word;
// bench.hpp: detail::synthetic_case, predict_gate_units), compiled against
// integration/locpir/gate_engine.hpp and evaluated by the tfhe-b200 engine kind, i.e.
// real TFHE bootstrapping on the GPU through include/locpir_b200.h.
//
//   b200_ref_driver truth <80|128>                 gate truth tables + counters
//   b200_ref_driver synthetic <80|128> N l m [w]   synthetic_case + loc_pir, w workers
//   b200_ref_driver city <80|128> <file>           the 9-city table (acceptance.cpp:173-237)
//   b200_ref_driver refkey                          the same engine around a reference
//                                                   keygen(TlweParams::sec128(), 31) key
// Every mode prints one JSON line.  Built by integration/Makefile (this container only:
// the reference headers are read from /root/reference); the binary travels to the GPU box.
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "locpir/locpir.hpp"

using namespace locpir;

namespace {

std::string counters_json(const GateEngine& e)
{
    const GateCounterSnapshot s = e.counters().snapshot();
    std::ostringstream o;
    o << "{\"and\": " << s.and_gates << ", \"or\": " << s.or_gates << ", \"xor\": " << s.xor_gates
      << ", \"xnor\": " << s.xnor_gates << ", \"not\": " << s.not_gates
      << ", \"mux\": " << s.mux_gates << ", \"bootstrap_units\": " << s.bootstrap_units() << "}";
    return o.str();
}

int truth(int sec)
{
    GateEngine e = GateEngine::make_tfhe_b200(sec, 7, 8);
    std::ostringstream o;
    o << "{\"mode\": \"truth\", \"engine\": \"" << engine_kind_name(e.kind()) << "\", \"bits\": [";
    bool first = true;
    auto put = [&](bool b) {
        o << (first ? "" : ", ") << (b ? 1 : 0);
        first = false;
    };
    // AND, OR, XOR, XNOR over (a, b) in 00, 01, 10, 11; NOT; MUX(sel, a, b) over 8 rows
    std::vector<CipherBit> outs;
    for (int g = 0; g < 4; g++)
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 2; b++) {
                CipherBit x = e.encrypt(a), y = e.encrypt(b);
                outs.push_back(g == 0 ? e.hom_and(x, y) : g == 1 ? e.hom_or(x, y)
                               : g == 2 ? e.hom_xor(x, y) : e.hom_xnor(x, y));
            }
    for (int a = 0; a < 2; a++)
        outs.push_back(e.hom_not(e.encrypt(a)));
    for (int s = 0; s < 2; s++)
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 2; b++)
                outs.push_back(e.hom_mux(e.encrypt(s), e.encrypt(a), e.encrypt(b)));
    // constants, and a refresh (one uncounted bootstrap) of an encryption of 1
    outs.push_back(e.hom_and(e.constant(true), e.encrypt(true)));
    const bool refreshed = decrypt_bit(e.refresh(e.encrypt(true).sample()), e.secret_key());
    for (const CipherBit& c : outs)
        put(e.decrypt(c));
    o << "], \"refresh\": " << (refreshed ? 1 : 0) << ", \"counters\": " << counters_json(e)
      << "}";
    std::cout << o.str() << std::endl;
    return 0;
}

int synthetic(int sec, uint32_t N, int l, uint32_t m, unsigned workers)
{
    GateEngine e = GateEngine::make_tfhe_b200(sec, 11, 12);
    SecretKey sk = e.secret_key();
    NoiseSampler client(13, sk.params.sigma);
    detail::SyntheticCase c = detail::synthetic_case(N, static_cast<uint8_t>(l), m, e, &client, &sk);
    e.counters().reset();
    const ServiceCiphertext out = loc_pir(c.x, c.y, c.regions, e, workers);
    const uint64_t got = decrypt_service(out, e);
    const uint64_t got_sk = decrypt_service(out, sk);
    std::cout << "{\"mode\": \"synthetic\", \"N\": " << N << ", \"l\": " << l << ", \"m\": " << m
              << ", \"workers\": " << workers << ", \"got\": " << got << ", \"got_sk\": " << got_sk
              << ", \"expected\": " << c.expected << ", \"units\": "
              << e.counters().snapshot().bootstrap_units()
              << ", \"predicted_units\": " << predict_gate_units(N, static_cast<uint8_t>(l), m)
              << ", \"counters\": " << counters_json(e) << "}" << std::endl;
    return 0;
}

// file: "boxes <4R ints>\nservices <R ints>\nbits <m>\nqueries <2Q ints>\nexpected <Q ints>"
int city(int sec, const char* path)
{
    std::ifstream in(path);
    std::map<std::string, std::vector<int64_t>> d;
    std::string line;
    while (std::getline(in, line)) {
        std::istringstream ls(line);
        std::string key;
        ls >> key;
        int64_t v;
        while (ls >> v)
            d[key].push_back(v);
    }
    const auto& bx = d["boxes"];
    const uint32_t R = static_cast<uint32_t>(bx.size() / 4), m = static_cast<uint32_t>(d["bits"].at(0));
    const FixedPointFormat fmt{9, 7};
    GateEngine e = GateEngine::make_tfhe_b200(sec, 31, 32);
    const SecretKey sk = e.secret_key();
    NoiseSampler client(33, sk.params.sigma);
    // services through the reference's zero-sample sheet flow (circuits.hpp:46-146)
    ZeroSampleSheet sheet = ZeroSampleSheet::generate(sk, R, m, client);
    std::vector<uint64_t> values(d["services"].begin(), d["services"].end());
    std::vector<ServiceCiphertext> svc = preprocess_services(values, sheet, m);
    std::vector<EncodedRegion> regions(R);
    auto word = [&](int64_t g) { return constant_word(PlainWord::from_integer(g, fmt), e); };
    for (uint32_t r = 0; r < R; r++)
        regions[r] = {word(bx[4 * r]), word(bx[4 * r + 1]), word(bx[4 * r + 2]), word(bx[4 * r + 3]),
                      std::move(svc[r]), r};
    const auto& qs = d["queries"];
    std::ostringstream o;
    o << "{\"mode\": \"city\", \"sec\": " << sec << ", \"got\": [";
    e.counters().reset();
    for (size_t q = 0; q < qs.size() / 2; q++) {
        const CipherWord x = encrypt_word(PlainWord::from_integer(qs[2 * q], fmt), sk, client);
        const CipherWord y = encrypt_word(PlainWord::from_integer(qs[2 * q + 1], fmt), sk, client);
        const ServiceCiphertext out = loc_pir(x, y, regions, e, 2);
        o << (q ? ", " : "") << decrypt_service(out, e);
    }
    o << "], \"expected\": [";
    for (size_t q = 0; q < d["expected"].size(); q++)
        o << (q ? ", " : "") << d["expected"][q];
    o << "], \"units\": " << e.counters().snapshot().bootstrap_units()
      << ", \"predicted_units_per_query\": " << predict_gate_units(R, fmt.total_bits(), m) << "}";
    std::cout << o.str() << std::endl;
    return 0;
}

int refkey()
{
    // a reference key and the reference's sec128 noise level
    const SecretKey sk = keygen(TlweParams::sec128(), 31);
    GateEngine e = GateEngine::make_tfhe_b200(sk, 31, 32);
    NoiseSampler client(33, sk.params.sigma);
    int wrong = 0, total = 0;
    for (int a = 0; a < 2; a++)
        for (int b = 0; b < 2; b++) {
            const CipherBit x(encrypt_bit(a, sk, client)), y(encrypt_bit(b, sk, client));
            wrong += e.decrypt(e.hom_xor(x, y)) != (a != b);
            wrong += e.decrypt(e.hom_and(x, y)) != (a && b);
            total += 2;
        }
    const PlainWord w1 = PlainWord::from_integer(-5, detail::format_for_length(8));
    const PlainWord w2 = PlainWord::from_integer(17, detail::format_for_length(8));
    const CipherBit lt = hom_less(encrypt_word(w1, sk, client), encrypt_word(w2, sk, client), e);
    wrong += !decrypt_bit(lt.sample(), sk);
    total++;
    std::cout << "{\"mode\": \"refkey\", \"n\": " << e.params().n << ", \"wrong\": " << wrong
              << ", \"total\": " << total << ", \"counters\": " << counters_json(e) << "}"
              << std::endl;
    return 0;
}

}  // namespace

int main(int argc, char** argv)
{
    try {
        const std::string mode = argc > 1 ? argv[1] : "";
        if (mode == "truth" && argc > 2)
            return truth(std::stoi(argv[2]));
        if (mode == "synthetic" && argc > 5)
            return synthetic(std::stoi(argv[2]), std::stoul(argv[3]), std::stoi(argv[4]),
                             std::stoul(argv[5]), argc > 6 ? std::stoul(argv[6]) : 1);
        if (mode == "city" && argc > 3)
            return city(std::stoi(argv[2]), argv[3]);
        if (mode == "refkey")
            return refkey();
        std::cerr << "usage: b200_ref_driver truth|synthetic|city|refkey ...\n";
        return 2;
    } catch (const std::exception& ex) {
        std::cout << "{\"error\": \"" << ex.what() << "\"}" << std::endl;
        return 1;
    }
}
