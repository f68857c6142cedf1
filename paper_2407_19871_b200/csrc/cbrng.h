/* cbrng.h -- counter-based client randomness, defined identically for the CPU oracle
 * (gcc, -ffp-contract=off) and the device (nvcc): SURVEY §8(f4) "a device RNG would break
 * seeded parity, so do it only with a counter-based RNG defined identically on the CPU".
 *
 * Philox4x32-10 (Salmon et al., SC'11; published constants) gives 4 u32 per
 * (counter, key).  Sample s of a stream with seed S uses key (lo32 S, hi32 S):
 *   mask word i  = philox((s, i / 4, 0, 0))[i % 4]
 *   noise        = philox((s, 0, 1, 0)) -> u1 in (0, 1], u2 in [0, 1) (53-bit)
 *                  z = sqrt(-2 ln u1) cos(2 pi u2)  (Box-Muller), e = rint(z * alpha * 2^32)
 * ln and cos are evaluated with +, -, *, /, fma, sqrt and frexp only -- all correctly
 * rounded IEEE operations -- so CPU and GPU produce the same bits.  Not the reference's
 * mt19937_64 stream (torus.hpp:119-138): this is the flagged device-encryption mode. */
#ifndef LOCPIR_CBRNG_H
#define LOCPIR_CBRNG_H
#include <stdint.h>

#ifdef __CUDACC__
#define CB_FN static __host__ __device__ __forceinline__
#else
#include <math.h>
#define CB_FN static inline
#endif

#if defined(__CUDA_ARCH__)
#define CB_FMA(a, b, c) __fma_rn(a, b, c)
#define CB_MUL(a, b) __dmul_rn(a, b)
#define CB_ADD(a, b) __dadd_rn(a, b)
#define CB_SUB(a, b) __dsub_rn(a, b)
#define CB_DIV(a, b) __ddiv_rn(a, b)
#define CB_SQRT(a) __dsqrt_rn(a)
#define CB_RINT64(a) __double2ll_rn(a)
#define CB_MULHI(a, b) __umulhi(a, b)
#else
#define CB_FMA(a, b, c) fma(a, b, c)
#define CB_MUL(a, b) ((a) * (b))
#define CB_ADD(a, b) ((a) + (b))
#define CB_SUB(a, b) ((a) - (b))
#define CB_DIV(a, b) ((a) / (b))
#define CB_SQRT(a) sqrt(a)
#define CB_RINT64(a) llrint(a)
#define CB_MULHI(a, b) ((uint32_t)(((uint64_t)(a) * (uint64_t)(b)) >> 32))
#endif

CB_FN void cb_philox(const uint32_t ctr_in[4], uint64_t seed, uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; r++) {
        const uint32_t hi0 = CB_MULHI(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = CB_MULHI(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0;
        c1 = n1;
        c2 = n2;
        c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

/* exact frexp for positive normal doubles: x = m * 2^e, m in [0.5, 1) */
CB_FN double cb_frexp(double x, int* e)
{
    union {
        double d;
        uint64_t u;
    } v;
    v.d = x;
    const int be = (int)((v.u >> 52) & 0x7FF);
    *e = be - 1022;
    v.u = (v.u & 0x800FFFFFFFFFFFFFull) | (1022ull << 52);
    return v.d;
}

/* ln(u), u in (0, 1] normal: u = m 2^k, m in [sqrt(1/2), sqrt(2)), ln m = 2 atanh(s),
 * s = (m - 1)/(m + 1), |s| <= 0.1716: series to s^23 (error < 1e-18). */
CB_FN double cb_log(double u)
{
    int k;
    double m = cb_frexp(u, &k);
    if (m < 0.70710678118654752440) {
        m = CB_MUL(m, 2.0);
        k -= 1;
    }
    const double s = CB_DIV(CB_SUB(m, 1.0), CB_ADD(m, 1.0));
    const double s2 = CB_MUL(s, s);
    double p = 1.0 / 23.0;
    p = CB_FMA(p, s2, 1.0 / 21.0);
    p = CB_FMA(p, s2, 1.0 / 19.0);
    p = CB_FMA(p, s2, 1.0 / 17.0);
    p = CB_FMA(p, s2, 1.0 / 15.0);
    p = CB_FMA(p, s2, 1.0 / 13.0);
    p = CB_FMA(p, s2, 1.0 / 11.0);
    p = CB_FMA(p, s2, 1.0 / 9.0);
    p = CB_FMA(p, s2, 1.0 / 7.0);
    p = CB_FMA(p, s2, 1.0 / 5.0);
    p = CB_FMA(p, s2, 1.0 / 3.0);
    p = CB_FMA(p, s2, 1.0);
    const double lnm = CB_MUL(CB_MUL(2.0, s), p);
    return CB_FMA((double)k, 0.69314718055994530942, lnm);
}

/* cos(2 pi x), x in [0, 1): quadrant q = round(4x), theta = 2 pi (x - q/4) in [-pi/4, pi/4] */
CB_FN double cb_cos2pi(double x)
{
    const double q4 = CB_MUL(x, 4.0);
    int q = (int)q4;
    if (CB_SUB(q4, (double)q) >= 0.5)
        q += 1;
    const double th = CB_MUL(6.28318530717958647693, CB_SUB(x, CB_MUL((double)q, 0.25)));
    const double t2 = CB_MUL(th, th);
    /* cos / sin Taylor series to degree 20 / 21 (|theta| <= pi/4: error < 1e-19) */
    double c = 1.0 / 2432902008176640000.0;          /* 1/20! */
    c = CB_FMA(c, -t2, 1.0 / 6402373705728000.0);    /* 1/18! */
    c = CB_FMA(c, -t2, 1.0 / 20922789888000.0);      /* 1/16! */
    c = CB_FMA(c, -t2, 1.0 / 87178291200.0);         /* 1/14! */
    c = CB_FMA(c, -t2, 1.0 / 479001600.0);           /* 1/12! */
    c = CB_FMA(c, -t2, 1.0 / 3628800.0);             /* 1/10! */
    c = CB_FMA(c, -t2, 1.0 / 40320.0);
    c = CB_FMA(c, -t2, 1.0 / 720.0);
    c = CB_FMA(c, -t2, 1.0 / 24.0);
    c = CB_FMA(c, -t2, 0.5);
    c = CB_FMA(c, -t2, 1.0);
    double s = 1.0 / 51090942171709440000.0;         /* 1/21! */
    s = CB_FMA(s, -t2, 1.0 / 121645100408832000.0);  /* 1/19! */
    s = CB_FMA(s, -t2, 1.0 / 355687428096000.0);     /* 1/17! */
    s = CB_FMA(s, -t2, 1.0 / 1307674368000.0);       /* 1/15! */
    s = CB_FMA(s, -t2, 1.0 / 6227020800.0);          /* 1/13! */
    s = CB_FMA(s, -t2, 1.0 / 39916800.0);            /* 1/11! */
    s = CB_FMA(s, -t2, 1.0 / 362880.0);
    s = CB_FMA(s, -t2, 1.0 / 5040.0);
    s = CB_FMA(s, -t2, 1.0 / 120.0);
    s = CB_FMA(s, -t2, 1.0 / 6.0);
    s = CB_FMA(s, -t2, 1.0);
    s = CB_MUL(s, th);
    switch (q & 3) {
    case 0: return c;
    case 1: return -s;
    case 2: return -c;
    default: return s;
    }
}

/* 53-bit uniforms from two u32: (hi:27 | lo:26) * 2^-53 */
CB_FN double cb_u53(uint32_t a, uint32_t b)
{
    const uint64_t v = ((uint64_t)(a >> 5) << 26) | (uint64_t)(b >> 6);
    return CB_MUL((double)v, 1.0 / 9007199254740992.0);
}

/* Noise word of sample `index`: rint(z * alpha * 2^32) mod 2^32. */
CB_FN uint32_t cb_noise(uint64_t seed, uint32_t index, double alpha)
{
    const uint32_t ctr[4] = {index, 0u, 1u, 0u};
    uint32_t r[4];
    cb_philox(ctr, seed, r);
    const double u1 = CB_SUB(1.0, cb_u53(r[0], r[1])); /* (0, 1] */
    const double u2 = cb_u53(r[2], r[3]);               /* [0, 1) */
    const double z = CB_MUL(CB_SQRT(CB_MUL(-2.0, cb_log(u1))), cb_cos2pi(u2));
    return (uint32_t)(uint64_t)CB_RINT64(CB_MUL(CB_MUL(z, alpha), 4294967296.0));
}

/* Mask word i of sample `index`. */
CB_FN uint32_t cb_mask_word(uint64_t seed, uint32_t index, uint32_t i)
{
    const uint32_t ctr[4] = {index, i >> 2, 0u, 0u};
    uint32_t r[4];
    cb_philox(ctr, seed, r);
    return r[i & 3];
}

#endif
