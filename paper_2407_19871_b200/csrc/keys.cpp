// keys.cpp -- client-side key material and encryption for the B200 engine.
//
// Host-only, no GPU.  Randomness is exactly the reference NoiseSampler: a
// std::mt19937_64 and a fresh std::normal_distribution<double> per Gaussian draw,
// rounded to the nearest multiple of 2^-32 (torus.hpp:38-43, :119-138).  The LWE
// key is the reference keygen (torus.hpp:146-154); encryption is the reference
// encrypt_torus / encrypt_bit (torus.hpp:161-175).  The TRLWE key, bootstrapping
// key and key-switching key extend it (SURVEY.md §8(a'), DESIGN.md "key
// derivation"): all derived from one seed through the reference's fork-lane
// mixer child_seed (gate_engine.hpp:601-607).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "../../include/locpir_b200.h"

namespace {

struct NoiseSampler {
    NoiseSampler(uint64_t seed, double sigma) : rng(seed), sigma(sigma) {}
    uint32_t uniform() { return static_cast<uint32_t>(rng()); }
    uint32_t gaussian()
    {
        if (sigma == 0.0)
            return 0;
        std::normal_distribution<double> dist(0.0, sigma);
        const double x = dist(rng);
        const double frac = x - std::floor(x);
        return static_cast<uint32_t>(static_cast<uint64_t>(std::llround(frac * 4294967296.0)));
    }
    std::mt19937_64 rng;
    double sigma;
};

uint64_t child_seed(uint64_t seed, uint64_t lane)
{
    uint64_t x = seed + 0x9e3779b97f4a7c15ull * (lane + 1);
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

bool valid(const locpir_b200_params* p)
{
    return p && p->n > 0 && p->n <= 1023 && p->N == 1024 && p->k == 1 && p->bk_l >= 1 &&
           p->bk_l * p->bk_bgbit <= 31 && p->ks_t * p->ks_basebit == 16 && p->ks_basebit == 2;
}

void encrypt_torus(uint32_t mu, const uint8_t* key, uint32_t n, NoiseSampler& s, uint32_t* out)
{
    uint32_t body = mu + s.gaussian();
    for (uint32_t i = 0; i < n; i++) {
        out[i] = s.uniform();
        if (key[i])
            body += out[i];
    }
    out[n] = body;
}

}  // namespace

extern "C" {

int locpir_b200_params_default(int security_bits, locpir_b200_params* out)
{
    if (!out)
        return LOCPIR_B200_EINVAL;
    if (security_bits == 80)
        *out = {500, 1024, 1, 2, 10, 8, 2, 2.44e-5, 7.18e-9};
    else if (security_bits == 128)
        *out = {630, 1024, 1, 3, 7, 8, 2, std::ldexp(1.0, -15), std::ldexp(1.0, -25)};
    else
        return LOCPIR_B200_EINVAL;
    return LOCPIR_B200_OK;
}

size_t locpir_b200_bk_words(const locpir_b200_params* p)
{
    return valid(p) ? (size_t)p->n * (p->k + 1) * p->bk_l * (p->k + 1) * p->N : 0;
}

size_t locpir_b200_ksk_words(const locpir_b200_params* p)
{
    return valid(p) ? (size_t)p->N * p->ks_t * ((1u << p->ks_basebit) - 1) * (p->n + 1) : 0;
}

static int keygen_impl(const locpir_b200_params* p, uint64_t seed, const uint8_t* lwe_key_in,
                       uint8_t* lwe_key_out, uint8_t* trlwe_key_out, uint32_t* bk_out,
                       uint32_t* ksk_out);

int locpir_b200_keygen(const locpir_b200_params* p, uint64_t seed, uint8_t* lwe_key_out,
                       uint8_t* trlwe_key_out, uint32_t* bk_out, uint32_t* ksk_out)
{
    return keygen_impl(p, seed, nullptr, lwe_key_out, trlwe_key_out, bk_out, ksk_out);
}

int locpir_b200_keygen_with_lwe_key(const locpir_b200_params* p, uint64_t seed,
                                    const uint8_t* lwe_key, uint8_t* trlwe_key_out,
                                    uint32_t* bk_out, uint32_t* ksk_out)
{
    if (!lwe_key)
        return LOCPIR_B200_EINVAL;
    for (uint32_t i = 0; valid(p) && i < p->n; i++)
        if (lwe_key[i] > 1)
            return LOCPIR_B200_EINVAL;
    return keygen_impl(p, seed, lwe_key, nullptr, trlwe_key_out, bk_out, ksk_out);
}

static int keygen_impl(const locpir_b200_params* p, uint64_t seed, const uint8_t* lwe_key_in,
                       uint8_t* lwe_key_out, uint8_t* trlwe_key_out, uint32_t* bk_out,
                       uint32_t* ksk_out)
{
    if (!valid(p))
        return LOCPIR_B200_EINVAL;
    const uint32_t n = p->n, N = p->N, l = p->bk_l, rows = 2 * l;
    std::vector<uint8_t> s(n), z(N);
    if (lwe_key_in) {
        std::memcpy(s.data(), lwe_key_in, n);
    } else {
        std::mt19937_64 rng(seed);  // torus.hpp:149-152
        for (auto& b : s)
            b = static_cast<uint8_t>(rng() & 1);
    }
    {
        std::mt19937_64 rng(child_seed(seed, 1));
        for (auto& b : z)
            b = static_cast<uint8_t>(rng() & 1);
    }
    if (lwe_key_out)
        std::memcpy(lwe_key_out, s.data(), n);
    if (trlwe_key_out)
        std::memcpy(trlwe_key_out, z.data(), N);

    if (bk_out) {
        // draws are sequential (one stream); the negacyclic products A*z run in parallel
        NoiseSampler smp(child_seed(seed, 2), p->alpha_bk);
        const size_t polys = (size_t)n * rows;
        for (size_t q = 0; q < polys; q++) {
            uint32_t* A = bk_out + (q * 2 + 0) * N;
            uint32_t* B = bk_out + (q * 2 + 1) * N;
            for (uint32_t j = 0; j < N; j++)
                A[j] = smp.uniform();
            for (uint32_t j = 0; j < N; j++)
                B[j] = smp.gaussian();
        }
        std::vector<uint32_t> zi;
        for (uint32_t m = 0; m < N; m++)
            if (z[m])
                zi.push_back(m);
        const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        std::vector<std::thread> th;
        for (unsigned w = 0; w < nt; w++)
            th.emplace_back([&, w] {
                for (size_t q = w; q < polys; q += nt) {
                    const uint32_t* A = bk_out + (q * 2 + 0) * N;
                    uint32_t* B = bk_out + (q * 2 + 1) * N;
                    for (uint32_t m : zi) {  // B += X^m * A (negacyclic)
                        for (uint32_t j = 0; j < m; j++)
                            B[j] -= A[j - m + N];
                        for (uint32_t j = m; j < N; j++)
                            B[j] += A[j - m];
                    }
                    const uint32_t i = (uint32_t)(q / rows), r = (uint32_t)(q % rows);
                    const uint32_t c = r / l, lev = r % l;
                    if (s[i]) {
                        const uint32_t h = 1u << (32 - (lev + 1) * p->bk_bgbit);
                        (c == 0 ? bk_out[(q * 2 + 0) * N] : B[0]) += h;
                    }
                }
            });
        for (auto& x : th)
            x.join();
    }
    if (ksk_out) {
        NoiseSampler smp(child_seed(seed, 3), p->alpha_in);
        const uint32_t base = 1u << p->ks_basebit;
        uint32_t* out = ksk_out;
        for (uint32_t i = 0; i < N; i++)
            for (uint32_t j = 0; j < p->ks_t; j++)
                for (uint32_t h = 1; h < base; h++) {
                    const uint32_t mu = (h * z[i]) << (32 - (j + 1) * p->ks_basebit);
                    encrypt_torus(mu, s.data(), n, smp, out);
                    out += n + 1;
                }
    }
    return LOCPIR_B200_OK;
}

int locpir_b200_encrypt_bits(const locpir_b200_params* p, const uint8_t* lwe_key, uint64_t seed,
                             const uint8_t* bits, uint64_t count, uint32_t* out)
{
    if (!valid(p) || !lwe_key || (count && (!bits || !out)))
        return LOCPIR_B200_EINVAL;
    NoiseSampler smp(seed, p->alpha_in);
    for (uint64_t i = 0; i < count; i++)
        encrypt_torus(bits[i] ? 0x20000000u : 0xE0000000u, lwe_key, p->n, smp,
                      out + i * (p->n + 1));
    return LOCPIR_B200_OK;
}

int locpir_b200_decrypt_bits(const locpir_b200_params* p, const uint8_t* lwe_key,
                             const uint32_t* cts, uint64_t count, uint8_t* bits_out)
{
    if (!valid(p) || !lwe_key || (count && (!cts || !bits_out)))
        return LOCPIR_B200_EINVAL;
    const uint32_t n = p->n;
    for (uint64_t g = 0; g < count; g++) {
        const uint32_t* ct = cts + g * (n + 1);
        uint32_t acc = ct[n];
        for (uint32_t i = 0; i < n; i++)
            if (lwe_key[i])
                acc -= ct[i];
        bits_out[g] = acc <= 0x80000000u;
    }
    return LOCPIR_B200_OK;
}

}  // extern "C"
