/*
 * tfhe_oracle.c -- CPU ORACLE (test infrastructure only; see tfhe_oracle.h).
 *
 * Compile with -ffp-contract=off: every floating-point rounding below is
 * explicit (fma() where a fused multiply-add is meant), because the B200
 * kernels reproduce this arithmetic bit-for-bit.
 */
#include "tfhe_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* mt19937_64 (the engine behind the reference NoiseSampler, torus.hpp:136)  */
/* ------------------------------------------------------------------------ */
#define MT_NN 312
#define MT_MM 156
#define MT_MATRIX_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

void or_mt64_seed(or_mt64* g, uint64_t seed)
{
    g->mt[0] = seed;
    for (int i = 1; i < MT_NN; i++)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->mti = MT_NN;
}

uint64_t or_mt64_next(or_mt64* g)
{
    static const uint64_t mag01[2] = {0ULL, MT_MATRIX_A};
    uint64_t x;
    if (g->mti >= MT_NN) {
        int i;
        for (i = 0; i < MT_NN - MT_MM; i++) {
            x = (g->mt[i] & MT_UM) | (g->mt[i + 1] & MT_LM);
            g->mt[i] = g->mt[i + MT_MM] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        for (; i < MT_NN - 1; i++) {
            x = (g->mt[i] & MT_UM) | (g->mt[i + 1] & MT_LM);
            g->mt[i] = g->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        x = (g->mt[MT_NN - 1] & MT_UM) | (g->mt[0] & MT_LM);
        g->mt[MT_NN - 1] = g->mt[MT_MM - 1] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        g->mti = 0;
    }
    x = g->mt[g->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* ------------------------------------------------------------------------ */
/* NoiseSampler (torus.hpp:119-138).  The reference constructs a fresh       */
/* std::normal_distribution<double> per draw (torus.hpp:129), so libstdc++'s */
/* Marsaglia polar method runs once per draw and its cached second value is  */
/* discarded.  generate_canonical<double,53> over a 64-bit engine takes one  */
/* engine output: u / 2^64, clamped below 1.                                 */
/* ------------------------------------------------------------------------ */
void or_sampler_init(or_sampler* s, uint64_t seed, double sigma)
{
    or_mt64_seed(&s->rng, seed);
    s->sigma = sigma;
}

uint32_t or_sampler_uniform(or_sampler* s) { return (uint32_t)or_mt64_next(&s->rng); }

static double canonical(or_mt64* g)
{
    double sum = (double)or_mt64_next(g);
    double ret = sum / 18446744073709551616.0;
    if (ret >= 1.0)
        ret = nextafter(1.0, 0.0);
    return ret;
}

double or_gaussian_double(or_sampler* s)
{
    double x, y, r2;
    do {
        x = 2.0 * canonical(&s->rng) - 1.0;
        y = 2.0 * canonical(&s->rng) - 1.0;
        r2 = x * x + y * y;
    } while (r2 > 1.0 || r2 == 0.0);
    const double mult = sqrt(-2.0 * log(r2) / r2);
    const double ret = y * mult;
    return ret * s->sigma + 0.0;
}

uint32_t or_torus_from_double(double x)
{
    double frac = x - floor(x);
    return (uint32_t)(uint64_t)llround(frac * 4294967296.0);
}

uint32_t or_sampler_gaussian(or_sampler* s)
{
    if (s->sigma == 0.0)
        return 0;
    return or_torus_from_double(or_gaussian_double(s));
}

uint64_t or_child_seed(uint64_t seed, uint64_t lane)
{
    uint64_t x = seed + 0x9e3779b97f4a7c15ULL * (lane + 1);
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* ------------------------------------------------------------------------ */
/* LWE layer (torus.hpp:146-222)                                             */
/* ------------------------------------------------------------------------ */
void or_keygen(uint32_t n, uint64_t seed, uint8_t* bits)
{
    or_mt64 g;
    or_mt64_seed(&g, seed);
    for (uint32_t i = 0; i < n; i++)
        bits[i] = (uint8_t)(or_mt64_next(&g) & 1);
}

void or_encrypt_torus(uint32_t mu, const uint8_t* key, uint32_t n, or_sampler* s, uint32_t* out)
{
    /* torus.hpp:161-170: body = mu + gaussian first, then mask draws */
    uint32_t body = mu + or_sampler_gaussian(s);
    for (uint32_t i = 0; i < n; i++) {
        out[i] = or_sampler_uniform(s);
        if (key[i])
            body += out[i];
    }
    out[n] = body;
}

void or_encrypt_bit(int bit, const uint8_t* key, uint32_t n, or_sampler* s, uint32_t* out)
{
    or_encrypt_torus(bit ? 0x20000000u : 0xE0000000u, key, n, s, out); /* torus.hpp:52-55 */
}

uint32_t or_phase(const uint32_t* ct, const uint8_t* key, uint32_t n)
{
    uint32_t acc = ct[n];
    for (uint32_t i = 0; i < n; i++)
        if (key[i])
            acc -= ct[i];
    return acc;
}

int or_decrypt_bit(const uint32_t* ct, const uint8_t* key, uint32_t n)
{
    return or_phase(ct, key, n) <= 0x80000000u; /* torus.hpp:191-194 */
}

void or_bootstrap_standin(const uint32_t* ct, const uint8_t* key, uint32_t n, or_sampler* s,
                          uint32_t* out)
{
    uint32_t p = or_phase(ct, key, n);
    int bit = p != 0 && p <= 0x80000000u; /* gate_engine.hpp:117-123 */
    or_encrypt_bit(bit, key, n, s, out);
}

/* ------------------------------------------------------------------------ */
/* TFHE parameters                                                           */
/* ------------------------------------------------------------------------ */
void or_params_default(int level, or_params* p)
{
    if (level == 80) {
        or_params q = {500, 1024, 1, 2, 10, 8, 2, 2.44e-5, 7.18e-9};
        *p = q;
    } else {
        or_params q = {630, 1024, 1, 3, 7, 8, 2, 0.0, 0.0};
        q.alpha_in = ldexp(1.0, -15);
        q.alpha_bk = ldexp(1.0, -25);
        *p = q;
    }
}

size_t or_bk_words(const or_params* p)
{
    return (size_t)p->n * (p->k + 1) * p->l * (p->k + 1) * p->N;
}

size_t or_ksk_words(const or_params* p)
{
    return (size_t)p->N * p->t * ((1u << p->basebit) - 1) * (p->n + 1);
}

/* ------------------------------------------------------------------------ */
/* Negacyclic FP64 transform (N = 1024 -> M = 512 complex points).           */
/* This is the arithmetic contract the B200 kernels execute operation for     */
/* operation (paper_2407_19871_b200/csrc/fft.cuh); TFHE's own FFT is absent   */
/* from /root/reference (parity unpinned, anchored on FFT == exact product).  */
/*                                                                            */
/* forward: a_j = d_j + i d_{j+M} (integers).  Evaluates P(Y) = sum a_j Y^j   */
/*   at the M roots of Y^M = i, i.e. Z_k = sum_j a_j psi^j W^{jk}             */
/*   (psi = e^{i pi/N}, W = e^{2 pi i/M}): the negacyclic twist is absorbed   */
/*   into the twiddles.  Cooley-Tukey recursion P mod (Y^{2h} - c) ->          */
/*   P mod (Y^h -+ r), r^2 = c: butterfly (u, v) -> (u + r v, u - r v).        */
/*   Tree node v = 2^s + b (stage s, block b) has modulus Y^{2h} - psi^E[v],   */
/*   E[1] = N/2, children E[v]/2 and E[v]/2 + N (mod 2N); twiddle             */
/*   r = psi^(E[v]/2).  Output slot b holds Z_{bitrev9(b)}.                   */
/* inverse: plain inverse DFT, radix-2 DIT, bit-reversed in -> natural out,   */
/*   twiddles conj(W^e), then the untwist conj(TW[j]) (TW = factored psi^j).  */
/*   The 1/M scale is folded into the frequency-domain BK (exact).            */
/*                                                                            */
/* Butterfly forms (every op rounds once, no contraction beyond the fma()s):  */
/*   CT(c, t):   w = c (1 + i t);  s = (fma(-vi, t, vr), fma(vr, t, vi));     */
/*               u' = (fma(c, sr, ur), fma(c, si, ui));                       */
/*               v' = (fma(-c, sr, ur), fma(-c, si, ui))        [6 fma]       */
/*   a rotation v -> i v or -i v (exact) may precede it;                      */
/*   STD(w):     t = cmul(v, w); u' = u + t; v' = u - t          [8 ops]      */
/*   trivial:    w = 1 or w = -i                                 [4 adds]     */
/* Which form each butterfly uses follows the GPU's 8 x 8 x 8 register layout */
/* (three passes of three stages): a stage's twiddle is a per-thread register */
/* value at the first stage of a pass and a register value times a compile-   */
/* time rotation at the other two (or_fwd_rule / or_inv_rule below).          */
/* ------------------------------------------------------------------------ */
typedef struct {
    double re, im;
} cplx;

static inline cplx cmul(cplx x, cplx w)
{
    cplx r;
    r.re = fma(x.re, w.re, -(x.im * w.im));
    r.im = fma(x.re, w.im, x.im * w.re);
    return r;
}

#define OR_M 512
#define OR_N 1024

typedef struct {
    int ready;
    double fc[OR_M], ft[OR_M];     /* forward twiddle base per tree node v (c, tan) */
    double W[OR_M / 2][2];         /* W^e, e < M/2, W[e + M/4] = i W[e] exactly */
    double ic[OR_M / 4], it[OR_M / 4]; /* inverse base (cos, tan) of W^e, e < M/4 */
    double TW[OR_M][2];            /* factored twist psi^j */
} fft2_tab;

static pthread_mutex_t g_tab_lock = PTHREAD_MUTEX_INITIALIZER;
static fft2_tab g_tab;

/* cos / tan of pi * num / den, rounded from long double (the product computes its
 * tables with the same libm calls) */
static void ct_of(long num, long den, double* c, double* t)
{
    const long double pi = 3.141592653589793238462643383279502884L;
    if (num == 0) {
        *c = 1.0;
        *t = 0.0;
        return;
    }
    if (4 * num == den) { /* pi/4: tan = 1 exactly */
        *c = (double)cosl(pi / 4.0L);
        *t = 1.0;
        return;
    }
    const long double th = pi * (long double)num / (long double)den;
    *c = (double)cosl(th);
    *t = (double)tanl(th);
}

void or_fft2_make_tables(double* fc, double* ft, double* W, double* ic, double* it, double* TW)
{
    const uint32_t M = OR_M, N = OR_N;
    uint32_t E[2 * OR_M];
    E[1] = N / 2;
    for (uint32_t v = 1; v < M; v++) {
        E[2 * v] = (E[v] / 2) % (2 * N);
        E[2 * v + 1] = (E[v] / 2 + N) % (2 * N);
    }
    fc[0] = ft[0] = 0.0;
    for (uint32_t v = 1; v < M; v++) /* twiddle psi^(E/2): angle pi (E/2) / N */
        ct_of((long)(E[v] / 2), (long)N, &fc[v], &ft[v]);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (uint32_t e = 0; e < M / 4; e++) {
        double re = 1.0, im = 0.0;
        if (e) {
            re = (double)cosl(2.0L * pi * (long double)e / (long double)M);
            im = (double)sinl(2.0L * pi * (long double)e / (long double)M);
        }
        W[2 * e] = re;
        W[2 * e + 1] = im;
        W[2 * (e + M / 4)] = -im;
        W[2 * (e + M / 4) + 1] = re;
        ct_of(2 * (long)e, (long)M, &ic[e], &it[e]);
    }
    /* twist psi^j in the factored form the GPU forms on the fly: TW[j] =
     * cmul(psi^(j mod 64), psi^(j - j mod 64)) with both factors rounded first */
    for (uint32_t j = 0; j < M; j++) {
        TW[2 * j] = j == 0 ? 1.0 : cos(3.14159265358979323846 * (double)j / (double)N);
        TW[2 * j + 1] = j == 0 ? 0.0 : sin(3.14159265358979323846 * (double)j / (double)N);
    }
    for (uint32_t j = M; j-- > 0;) { /* descending: factors j & 63, j & ~63 are still exact */
        const uint32_t lo = j & 63u, hi = j & ~63u;
        if (lo && hi) {
            const double xr = TW[2 * lo], xi = TW[2 * lo + 1];
            const double wr = TW[2 * hi], wi = TW[2 * hi + 1];
            TW[2 * j] = fma(xr, wr, -(xi * wi));
            TW[2 * j + 1] = fma(xr, wi, xi * wr);
        }
    }
}

static const fft2_tab* get_tab(uint32_t N)
{
    if (N != OR_N)
        return NULL;
    pthread_mutex_lock(&g_tab_lock);
    if (!g_tab.ready) {
        or_fft2_make_tables(g_tab.fc, g_tab.ft, &g_tab.W[0][0], g_tab.ic, g_tab.it, &g_tab.TW[0][0]);
        g_tab.ready = 1;
    }
    pthread_mutex_unlock(&g_tab_lock);
    return &g_tab;
}

/* kept for the API: W (N/4 complex), TW, UT = conj(TW) (no 1/M: folded into the BK) */
void or_fft_tables(uint32_t N, double* W, double* TW, double* UT)
{
    const fft2_tab* t = get_tab(N);
    if (!t)
        return;
    memcpy(W, t->W, sizeof(t->W));
    memcpy(TW, t->TW, sizeof(t->TW));
    for (uint32_t j = 0; j < OR_M; j++) {
        UT[2 * j] = t->TW[j][0];
        UT[2 * j + 1] = -t->TW[j][1];
    }
}

/* rot: 0 none, 1 multiply v by i, 3 multiply v by -i */
static inline void bf_ct(double* ur, double* ui, double* vr, double* vi, double c, double t,
                         int rot)
{
    double xr = *vr, xi = *vi;
    if (rot == 1) {
        const double tmp = xr;
        xr = -xi;
        xi = tmp;
    } else if (rot == 3) {
        const double tmp = xr;
        xr = xi;
        xi = -tmp;
    }
    const double sr = fma(-xi, t, xr), si = fma(xr, t, xi);
    const double a = *ur, b = *ui;
    *ur = fma(c, sr, a);
    *ui = fma(c, si, b);
    *vr = fma(-c, sr, a);
    *vi = fma(-c, si, b);
}

static inline void bf_std(double* ur, double* ui, double* vr, double* vi, double wr, double wi)
{
    cplx v = {*vr, *vi}, w = {wr, wi};
    const cplx t = cmul(v, w);
    const double a = *ur, b = *ui;
    *ur = a + t.re;
    *ui = b + t.im;
    *vr = a - t.re;
    *vi = b - t.im;
}

static inline void bf_1(double* ur, double* ui, double* vr, double* vi)
{
    const double a = *ur, b = *ui, c = *vr, d = *vi;
    *ur = a + c;
    *ui = b + d;
    *vr = a - c;
    *vi = b - d;
}

static inline void bf_mi(double* ur, double* ui, double* vr, double* vi) /* w = -i */
{
    const double a = *ur, b = *ui, c = *vi, d = -*vr; /* -i v = (vi, -vr) */
    *ur = a + c;
    *ui = b + d;
    *vr = a - c;
    *vi = b - d;
}

/* forward rule: at stage s, block b uses node v = 2^s + b's own twiddle, except at
 * stages s % 3 != 0 where an odd block uses its even sibling's twiddle after v -> i v
 * (the sibling bit is a register bit of the GPU layout there) */
static void fwd_soa(const fft2_tab* T, double* zr, double* zi)
{
    const uint32_t M = OR_M;
    for (uint32_t s = 0; s < 9; s++) {
        const uint32_t h = M >> (s + 1);
        for (uint32_t b = 0; b < (1u << s); b++) {
            const int sib = (s % 3 != 0) && (b & 1);
            const uint32_t v = (1u << s) + b - (sib ? 1 : 0);
            const double c = T->fc[v], t = T->ft[v];
            const uint32_t o = 2 * h * b;
            for (uint32_t j = 0; j < h; j++)
                bf_ct(&zr[o + j], &zi[o + j], &zr[o + j + h], &zi[o + j + h], c, t, sib ? 1 : 0);
        }
    }
}

/* inverse rule (stage half-size h = 1 .. 256, butterfly (j, j + h), twiddle conj(W^e),
 * e = j * (M/2) / h):
 *   h <= 4, e in {0, M/4}: trivial;  h in {8, 64} (first stage of a GPU pass): STD with
 *   the per-thread value conj(W[e]);  otherwise CT with the base e mod M/4 (conj: tan
 *   negated), after v -> -i v when e >= M/4. */
static void inv_soa(const fft2_tab* T, double* zr, double* zi)
{
    const uint32_t M = OR_M;
    for (uint32_t h = 1; h < M; h <<= 1) {
        const uint32_t step = (M / 2) / h;
        for (uint32_t o = 0; o < M; o += 2 * h)
            for (uint32_t j = 0; j < h; j++) {
                const uint32_t e = j * step;
                double *ur = &zr[o + j], *ui = &zi[o + j], *vr = &zr[o + j + h], *vi = &zi[o + j + h];
                if (h <= 4 && e == 0)
                    bf_1(ur, ui, vr, vi);
                else if (h <= 4 && e == M / 4)
                    bf_mi(ur, ui, vr, vi);
                else if (h == 8 || h == 64)
                    bf_std(ur, ui, vr, vi, T->W[e][0], -T->W[e][1]);
                else {
                    const uint32_t e0 = e % (M / 4);
                    bf_ct(ur, ui, vr, vi, T->ic[e0], -T->it[e0], e >= M / 4 ? 3 : 0);
                }
            }
    }
}

/* forward of integer digits: out = (re, im) pairs in slot order (unscaled) */
void or_fft_forward_i32(uint32_t N, const int32_t* in, double* out)
{
    const fft2_tab* t = get_tab(N);
    const uint32_t M = OR_M;
    double zr[OR_M], zi[OR_M];
    for (uint32_t j = 0; j < M; j++) {
        zr[j] = (double)in[j];
        zi[j] = (double)in[j + M];
    }
    fwd_soa(t, zr, zi);
    for (uint32_t j = 0; j < M; j++) {
        out[2 * j] = zr[j];
        out[2 * j + 1] = zi[j];
    }
}

/* inverse: untwist, round each coefficient to the nearest integer mod 2^32 and ADD it
 * into acc[N]; `in` (slot order) is the spectrum of a product with a 1/M-scaled BK */
/* diagnostic: max distance of an inverse output from the nearest integer before rounding
 * (the FFT rounding margin; coefficients are exact while it stays below 1/2) */
static double g_fft_err = 0.0;
static pthread_mutex_t g_err_lock = PTHREAD_MUTEX_INITIALIZER;
double or_fft_margin(int reset)
{
    pthread_mutex_lock(&g_err_lock);
    const double e = g_fft_err;
    if (reset)
        g_fft_err = 0.0;
    pthread_mutex_unlock(&g_err_lock);
    return e;
}

static void inverse_add_soa(const fft2_tab* t, double* zr, double* zi, uint32_t* acc)
{
    inv_soa(t, zr, zi);
    double emax = 0.0;
    for (uint32_t j = 0; j < OR_M; j++) {
        const cplx y = {zr[j], zi[j]};
        const cplx u = {t->TW[j][0], -t->TW[j][1]};
        const cplx w = cmul(y, u);
        emax = fmax(emax, fmax(fabs(w.re - rint(w.re)), fabs(w.im - rint(w.im))));
        acc[j] += (uint32_t)(uint64_t)llrint(w.re);
        acc[j + OR_M] += (uint32_t)(uint64_t)llrint(w.im);
    }
    if (emax > g_fft_err) {
        pthread_mutex_lock(&g_err_lock);
        if (emax > g_fft_err)
            g_fft_err = emax;
        pthread_mutex_unlock(&g_err_lock);
    }
}

void or_fft_inverse_add(uint32_t N, double* in, uint32_t* acc)
{
    const fft2_tab* t = get_tab(N);
    double zr[OR_M], zi[OR_M];
    for (uint32_t j = 0; j < OR_M; j++) {
        zr[j] = in[2 * j];
        zi[j] = in[2 * j + 1];
    }
    inverse_add_soa(t, zr, zi, acc);
}

void or_polymul_exact_add(uint32_t N, const int32_t* d, const uint32_t* b, uint32_t* acc)
{
    for (uint32_t m = 0; m < N; m++) {
        const uint32_t dm = (uint32_t)d[m];
        if (dm == 0)
            continue;
        /* X^m * b : coefficient j gets b[j-m] (j>=m) or -b[j-m+N] */
        for (uint32_t j = 0; j < m; j++)
            acc[j] -= dm * b[j - m + N];
        for (uint32_t j = m; j < N; j++)
            acc[j] += dm * b[j - m];
    }
}

/* ------------------------------------------------------------------------ */
/* Gadget decomposition: signed digits with the rounding offset               */
/* (x' = x + sum_p Bg/2 * 2^(32-p*Bgbit) + 2^(31 - l*Bgbit)).                 */
/* ------------------------------------------------------------------------ */
static uint32_t decomp_offset(const or_params* p)
{
    uint32_t off = 0;
    const uint32_t half = 1u << (p->bgbit - 1);
    for (uint32_t q = 1; q <= p->l; q++)
        off += half << (32 - q * p->bgbit);
    off += 1u << (31 - p->l * p->bgbit);
    return off;
}

void or_decompose(const or_params* p, const uint32_t* x, uint32_t level, int32_t* digits)
{
    const uint32_t off = decomp_offset(p);
    const uint32_t shift = 32 - (level + 1) * p->bgbit;
    const uint32_t mask = (1u << p->bgbit) - 1;
    const int32_t half = 1 << (p->bgbit - 1);
    for (uint32_t j = 0; j < p->N; j++)
        digits[j] = (int32_t)(((x[j] + off) >> shift) & mask) - half;
}

uint32_t or_mod_switch(uint32_t x, uint32_t N)
{
    uint32_t logN2 = 0;
    while ((1u << logN2) < 2 * N)
        logN2++;
    const uint32_t sh = 32 - logN2;
    return (uint32_t)(x + (1u << (sh - 1))) >> sh;
}

/* ------------------------------------------------------------------------ */
/* Key set                                                                   */
/* ------------------------------------------------------------------------ */
static void negacyclic_mul_binary_add(uint32_t N, const uint32_t* a, const uint8_t* z,
                                      uint32_t* acc)
{
    for (uint32_t m = 0; m < N; m++) {
        if (!z[m])
            continue;
        for (uint32_t j = 0; j < m; j++)
            acc[j] -= a[j - m + N];
        for (uint32_t j = m; j < N; j++)
            acc[j] += a[j - m];
    }
}

int or_keyset_generate(or_keyset* ks, const or_params* p, uint64_t seed)
{
    if (p->k != 1 || p->N < 16 || (p->N & (p->N - 1)))
        return -1;
    memset(ks, 0, sizeof(*ks));
    ks->p = *p;
    const uint32_t n = p->n, N = p->N, rows = (p->k + 1) * p->l;
    const uint32_t base = 1u << p->basebit;
    ks->lwe_key = (uint8_t*)malloc(n);
    ks->trlwe_key = (uint8_t*)malloc(N);
    ks->bk = (uint32_t*)malloc(sizeof(uint32_t) * or_bk_words(p));
    ks->ksk = (uint32_t*)malloc(sizeof(uint32_t) * or_ksk_words(p));
    ks->bk_fft = (double*)malloc(sizeof(double) * or_bk_words(p));
    ks->bk_fft_soa = (double*)malloc(sizeof(double) * or_bk_words(p));
    if (!ks->lwe_key || !ks->trlwe_key || !ks->bk || !ks->ksk || !ks->bk_fft || !ks->bk_fft_soa)
        return -2;

    /* LWE key: the reference keygen (torus.hpp:146-154) */
    or_keygen(n, seed, ks->lwe_key);
    /* TRLWE key: N binary coefficients from an independent lane */
    {
        or_mt64 g;
        or_mt64_seed(&g, or_child_seed(seed, 1));
        for (uint32_t j = 0; j < N; j++)
            ks->trlwe_key[j] = (uint8_t)(or_mt64_next(&g) & 1);
    }
    /* BK: n TRGSW encryptions of s_i; row (c, q) = TRLWE_z(0) + s_i * 2^(32-(q+1)Bgbit)
     * on component c.  Draw order per row: N uniform mask coefficients, then N
     * Gaussian noise coefficients. */
    {
        or_sampler s;
        or_sampler_init(&s, or_child_seed(seed, 2), p->alpha_bk);
        for (uint32_t i = 0; i < n; i++)
            for (uint32_t r = 0; r < rows; r++) {
                uint32_t* A = ks->bk + (((size_t)i * rows + r) * 2 + 0) * N;
                uint32_t* B = ks->bk + (((size_t)i * rows + r) * 2 + 1) * N;
                for (uint32_t j = 0; j < N; j++)
                    A[j] = or_sampler_uniform(&s);
                for (uint32_t j = 0; j < N; j++)
                    B[j] = or_sampler_gaussian(&s);
                negacyclic_mul_binary_add(N, A, ks->trlwe_key, B);
                const uint32_t c = r / p->l, q = r % p->l;
                const uint32_t h = 1u << (32 - (q + 1) * p->bgbit);
                if (ks->lwe_key[i]) {
                    if (c == 0)
                        A[0] += h;
                    else
                        B[0] += h;
                }
            }
    }
    /* KSK[i][j][h-1] = LWE_s(h * z_i * 2^(32-(j+1)basebit)) with the reference
     * encrypt_torus (torus.hpp:161-170). */
    {
        or_sampler s;
        or_sampler_init(&s, or_child_seed(seed, 3), p->alpha_in);
        uint32_t* out = ks->ksk;
        for (uint32_t i = 0; i < N; i++)
            for (uint32_t j = 0; j < p->t; j++)
                for (uint32_t h = 1; h < base; h++) {
                    const uint32_t mu = (h * ks->trlwe_key[i]) << (32 - (j + 1) * p->basebit);
                    or_encrypt_torus(mu, ks->lwe_key, n, &s, out);
                    out += n + 1;
                }
    }
    /* frequency-domain BK */
    {
        int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * N);
        const size_t polys = (size_t)n * rows * 2;
        for (size_t q = 0; q < polys; q++) {
            for (uint32_t j = 0; j < N; j++)
                tmp[j] = (int32_t)ks->bk[q * N + j];
            or_fft_forward_i32(N, tmp, ks->bk_fft + q * N);
            for (uint32_t f = 0; f < N; f++) /* 1/M folded into the key (exact) */
                ks->bk_fft[q * N + f] *= 1.0 / (double)(N / 2);
            for (uint32_t f = 0; f < N / 2; f++) {
                ks->bk_fft_soa[q * N + f] = ks->bk_fft[q * N + 2 * f];
                ks->bk_fft_soa[q * N + N / 2 + f] = ks->bk_fft[q * N + 2 * f + 1];
            }
        }
        free(tmp);
    }
    return 0;
}

void or_keyset_free(or_keyset* ks)
{
    free(ks->lwe_key);
    free(ks->trlwe_key);
    free(ks->bk);
    free(ks->ksk);
    free(ks->bk_fft);
    free(ks->bk_fft_soa);
    memset(ks, 0, sizeof(*ks));
}

/* ------------------------------------------------------------------------ */
/* Bootstrapping                                                             */
/* ------------------------------------------------------------------------ */
/* out = X^e * in, e in [0, 2N) */
static void poly_mul_xai(uint32_t N, uint32_t e, const uint32_t* in, uint32_t* out)
{
    if (e < N) {
        for (uint32_t j = 0; j < e; j++)
            out[j] = 0u - in[j - e + N];
        for (uint32_t j = e; j < N; j++)
            out[j] = in[j - e];
    } else {
        const uint32_t f = e - N;
        for (uint32_t j = 0; j < f; j++)
            out[j] = in[j - f + N];
        for (uint32_t j = f; j < N; j++)
            out[j] = 0u - in[j - f];
    }
}

int or_external_product(const or_keyset* ks, uint32_t i, const uint32_t* trlwe, int mode,
                        uint32_t* out)
{
    const or_params* p = &ks->p;
    const uint32_t N = p->N, M = N / 2, rows = (p->k + 1) * p->l;
    int32_t* dig = (int32_t*)malloc(sizeof(int32_t) * N);
    memset(out, 0, sizeof(uint32_t) * 2 * N);
    if (mode == ORACLE_EXACT) {
        for (uint32_t c = 0; c < 2; c++)
            for (uint32_t q = 0; q < p->l; q++) {
                or_decompose(p, trlwe + c * N, q, dig);
                const uint32_t r = c * p->l + q;
                for (uint32_t comp = 0; comp < 2; comp++)
                    or_polymul_exact_add(N, dig, ks->bk + (((size_t)i * rows + r) * 2 + comp) * N,
                                         out + comp * N);
            }
    } else {
        const fft2_tab* tab = get_tab(N);
        double Fr[512], Fi[512], Ar[2][512], Ai[2][512];
        memset(Ar, 0, sizeof(Ar));
        memset(Ai, 0, sizeof(Ai));
        for (uint32_t c = 0; c < 2; c++)
            for (uint32_t q = 0; q < p->l; q++) {
                or_decompose(p, trlwe + c * N, q, dig);
                for (uint32_t j = 0; j < M; j++) {
                    Fr[j] = (double)dig[j];
                    Fi[j] = (double)dig[j + M];
                }
                fwd_soa(tab, Fr, Fi);
                const uint32_t r = c * p->l + q;
                for (uint32_t comp = 0; comp < 2; comp++) {
                    const double* Br = ks->bk_fft_soa + (((size_t)i * rows + r) * 2 + comp) * N;
                    const double* Bi = Br + M;
                    double* ar = Ar[comp];
                    double* ai = Ai[comp];
                    for (uint32_t f = 0; f < M; f++) {
                        double re = fma(Fr[f], Br[f], ar[f]);
                        re = fma(-Fi[f], Bi[f], re);
                        double im = fma(Fr[f], Bi[f], ai[f]);
                        im = fma(Fi[f], Br[f], im);
                        ar[f] = re;
                        ai[f] = im;
                    }
                }
            }
        for (uint32_t comp = 0; comp < 2; comp++)
            inverse_add_soa(tab, Ar[comp], Ai[comp], out + comp * N);
    }
    free(dig);
    return 0;
}

int or_blind_rotate_acc(const or_keyset* ks, const uint32_t* lwe_in, uint32_t mu, int mode,
                        uint32_t steps, uint32_t* acc)
{
    const or_params* p = &ks->p;
    const uint32_t n = p->n, N = p->N;
    uint32_t* v = (uint32_t*)malloc(sizeof(uint32_t) * N);
    uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
    uint32_t* ext = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
    for (uint32_t j = 0; j < N; j++)
        v[j] = mu;
    const uint32_t bbar = or_mod_switch(lwe_in[n], N);
    memset(acc, 0, sizeof(uint32_t) * N);
    poly_mul_xai(N, (2 * N - bbar) % (2 * N), v, acc + N);
    for (uint32_t i = 0; i < n && i < steps; i++) {
        const uint32_t a = or_mod_switch(lwe_in[i], N);
        if (a == 0)
            continue;
        for (uint32_t c = 0; c < 2; c++) {
            poly_mul_xai(N, a, acc + c * N, tmp + c * N);
            for (uint32_t j = 0; j < N; j++)
                tmp[c * N + j] -= acc[c * N + j];
        }
        or_external_product(ks, i, tmp, mode, ext);
        for (uint32_t j = 0; j < 2 * N; j++)
            acc[j] += ext[j];
    }
    free(v);
    free(tmp);
    free(ext);
    return 0;
}

int or_blind_rotate_extract(const or_keyset* ks, const uint32_t* lwe_in, uint32_t mu, int mode,
                            uint32_t* out_N)
{
    const uint32_t N = ks->p.N;
    uint32_t* acc = (uint32_t*)malloc(sizeof(uint32_t) * 2 * N);
    or_blind_rotate_acc(ks, lwe_in, mu, mode, 0xFFFFFFFFu, acc);
    /* sample extraction at index 0 */
    out_N[0] = acc[0];
    for (uint32_t j = 1; j < N; j++)
        out_N[j] = 0u - acc[N - j];
    out_N[N] = acc[N];
    free(acc);
    return 0;
}

void or_keyswitch(const or_keyset* ks, const uint32_t* in_N, uint32_t* out_n)
{
    const or_params* p = &ks->p;
    const uint32_t n = p->n, N = p->N, base = 1u << p->basebit;
    const uint32_t prec = 1u << (32 - (1 + p->basebit * p->t));
    const uint32_t mask = base - 1;
    memset(out_n, 0, sizeof(uint32_t) * n);
    out_n[n] = in_N[N];
    for (uint32_t i = 0; i < N; i++) {
        const uint32_t abar = in_N[i] + prec;
        for (uint32_t j = 0; j < p->t; j++) {
            const uint32_t d = (abar >> (32 - (j + 1) * p->basebit)) & mask;
            if (!d)
                continue;
            const uint32_t* row = ks->ksk + (((size_t)i * p->t + j) * (base - 1) + (d - 1)) * (n + 1);
            for (uint32_t q = 0; q <= n; q++)
                out_n[q] -= row[q];
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Gates                                                                     */
/* ------------------------------------------------------------------------ */
static void lin2(uint32_t n, uint32_t off, int32_t ca, const uint32_t* a, int32_t cb,
                 const uint32_t* b, uint32_t* out)
{
    for (uint32_t q = 0; q <= n; q++)
        out[q] = (uint32_t)ca * a[q] + (uint32_t)cb * b[q];
    out[n] += off;
}

int or_gate(const or_keyset* ks, int kind, const uint32_t* a, const uint32_t* b,
            const uint32_t* c, int mode, uint32_t* out)
{
    const uint32_t n = ks->p.n, N = ks->p.N;
    const uint32_t MU = 0x20000000u;
    uint32_t* comb = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
    uint32_t* ext = (uint32_t*)malloc(sizeof(uint32_t) * (N + 1));
    int rc = 0;
    switch (kind) {
    case OR_GATE_AND: lin2(n, 0xE0000000u, 1, a, 1, b, comb); break;
    case OR_GATE_OR: lin2(n, 0x20000000u, 1, a, 1, b, comb); break;
    case OR_GATE_XOR: lin2(n, 0x40000000u, 2, a, 2, b, comb); break;
    case OR_GATE_XNOR: lin2(n, 0xC0000000u, -2, a, -2, b, comb); break;
    case OR_GATE_NAND: lin2(n, 0x20000000u, -1, a, -1, b, comb); break;
    case OR_GATE_NOR: lin2(n, 0xE0000000u, -1, a, -1, b, comb); break;
    case OR_GATE_ANDNY: lin2(n, 0xE0000000u, -1, a, 1, b, comb); break;
    case OR_GATE_ORNY: lin2(n, 0x20000000u, -1, a, 1, b, comb); break;
    case OR_GATE_MAJ:
        lin2(n, 0u, 1, a, 1, b, comb);
        for (uint32_t q = 0; q <= n; q++)
            comb[q] += c[q];
        break;
    case OR_GATE_XOR3:
        lin2(n, 0u, -2, a, -2, b, comb);
        for (uint32_t q = 0; q <= n; q++)
            comb[q] += (uint32_t)-2 * c[q];
        break;
    case OR_GATE_NOT:
        for (uint32_t q = 0; q <= n; q++)
            out[q] = 0u - a[q];
        goto done;
    case OR_GATE_MUX: {
        /* TFHE MUX: u1 = BR(-1/8 + s + a), u2 = BR(-1/8 - s + b), out = KS(u1 + u2 + 1/8) */
        uint32_t* ext2 = (uint32_t*)malloc(sizeof(uint32_t) * (N + 1));
        lin2(n, 0xE0000000u, 1, a, 1, b, comb);
        or_blind_rotate_extract(ks, comb, MU, mode, ext);
        lin2(n, 0xE0000000u, -1, a, 1, c, comb);
        or_blind_rotate_extract(ks, comb, MU, mode, ext2);
        for (uint32_t q = 0; q <= N; q++)
            ext[q] += ext2[q];
        ext[N] += 0x20000000u;
        or_keyswitch(ks, ext, out);
        free(ext2);
        goto done;
    }
    default: rc = -1; goto done;
    }
    or_blind_rotate_extract(ks, comb, MU, mode, ext);
    or_keyswitch(ks, ext, out);
done:
    free(comb);
    free(ext);
    return rc;
}

typedef struct {
    const or_keyset* ks;
    int kind, mode;
    const uint32_t *a, *b;
    uint32_t* out;
    uint64_t lo, hi;
    int rc;
} batch_job;

static void* batch_worker(void* arg)
{
    batch_job* j = (batch_job*)arg;
    const size_t w = j->ks->p.n + 1;
    for (uint64_t g = j->lo; g < j->hi; g++) {
        int rc = or_gate(j->ks, j->kind, j->a + g * w, j->b ? j->b + g * w : NULL, NULL, j->mode,
                         j->out + g * w);
        if (rc)
            j->rc = rc;
    }
    return NULL;
}

int or_gate_batch(const or_keyset* ks, int kind, const uint32_t* a, const uint32_t* b,
                  uint32_t* out, uint64_t count, int mode, int threads)
{
    if (threads < 1)
        threads = 1;
    if ((uint64_t)threads > count)
        threads = count ? (int)count : 1;
    batch_job* jobs = (batch_job*)calloc(threads, sizeof(batch_job));
    pthread_t* tid = (pthread_t*)calloc(threads, sizeof(pthread_t));
    const uint64_t chunk = (count + threads - 1) / threads; /* parallel.hpp:26-34 */
    for (int w = 0; w < threads; w++) {
        jobs[w].ks = ks;
        jobs[w].kind = kind;
        jobs[w].mode = mode;
        jobs[w].a = a;
        jobs[w].b = b;
        jobs[w].out = out;
        jobs[w].lo = (uint64_t)w * chunk < count ? (uint64_t)w * chunk : count;
        jobs[w].hi = jobs[w].lo + chunk < count ? jobs[w].lo + chunk : count;
    }
    for (int w = 1; w < threads; w++)
        pthread_create(&tid[w], NULL, batch_worker, &jobs[w]);
    batch_worker(&jobs[0]);
    int rc = jobs[0].rc;
    for (int w = 1; w < threads; w++) {
        pthread_join(tid[w], NULL);
        if (jobs[w].rc)
            rc = jobs[w].rc;
    }
    free(jobs);
    free(tid);
    return rc;
}

typedef struct {
    const or_keyset* ks;
    const or_gate_item* items;
    int mode;
    uint64_t lo, hi;
    int rc;
} list_job;

static void* list_worker(void* arg)
{
    list_job* j = (list_job*)arg;
    for (uint64_t g = j->lo; g < j->hi; g++) {
        const or_gate_item* it = &j->items[g];
        int rc = or_gate(j->ks, it->kind, it->a, it->b, it->c, j->mode, it->out);
        if (rc)
            j->rc = rc;
    }
    return NULL;
}

int or_gate_list(const or_keyset* ks, const or_gate_item* items, uint64_t count, int mode,
                 int threads)
{
    if (threads < 1)
        threads = 1;
    if ((uint64_t)threads > count)
        threads = count ? (int)count : 1;
    list_job* jobs = (list_job*)calloc(threads, sizeof(list_job));
    pthread_t* tid = (pthread_t*)calloc(threads, sizeof(pthread_t));
    const uint64_t chunk = (count + threads - 1) / threads;
    for (int w = 0; w < threads; w++) {
        jobs[w].ks = ks;
        jobs[w].items = items;
        jobs[w].mode = mode;
        jobs[w].lo = (uint64_t)w * chunk < count ? (uint64_t)w * chunk : count;
        jobs[w].hi = jobs[w].lo + chunk < count ? jobs[w].lo + chunk : count;
    }
    for (int w = 1; w < threads; w++)
        pthread_create(&tid[w], NULL, list_worker, &jobs[w]);
    list_worker(&jobs[0]);
    int rc = jobs[0].rc;
    for (int w = 1; w < threads; w++) {
        pthread_join(tid[w], NULL);
        if (jobs[w].rc)
            rc = jobs[w].rc;
    }
    free(jobs);
    free(tid);
    return rc;
}

/* ---- counter-based client encryption ------------------------------
 * The stream is DEFINED by paper_2407_19871_b200/csrc/cbrng.h (one definition for CPU and
 * GPU); the oracle evaluates it on the host so the device kernel can be checked bit for
 * bit.  Philox itself is pinned to its published known answers in the tests. */
#include "../paper_2407_19871_b200/csrc/cbrng.h"

void or_cb_philox(const uint32_t ctr[4], uint64_t seed, uint32_t out[4]) { cb_philox(ctr, seed, out); }
double or_cb_log(double u) { return cb_log(u); }
double or_cb_cos2pi(double x) { return cb_cos2pi(x); }
uint32_t or_cb_noise(uint64_t seed, uint32_t index, double alpha) { return cb_noise(seed, index, alpha); }

void or_cb_encrypt(const uint8_t* key, uint32_t n, uint64_t seed, uint32_t first_index,
                   const uint32_t* mus, uint64_t count, double alpha, uint32_t* out)
{
    for (uint64_t j = 0; j < count; j++) {
        const uint32_t idx = first_index + (uint32_t)j;
        uint32_t* o = out + j * (n + 1);
        uint32_t dot = 0;
        for (uint32_t i = 0; i < n; i++) {
            o[i] = cb_mask_word(seed, idx, i);
            dot += o[i] * (uint32_t)key[i];
        }
        o[n] = dot + mus[j] + cb_noise(seed, idx, alpha);
    }
}

/* ------------------------------------------------------------------------ */
/* Lane-batched FFT-mode gates (CPU baseline speed; same arithmetic)         */
/* ------------------------------------------------------------------------ */
/* or_gate_batch_simd: the FFT-mode gate of or_gate for VL ciphertexts at a time, one per
 * SIMD lane (VL = 8 with AVX-512, 4 with AVX2).  Every lane executes exactly the scalar
 * operation sequence (the same fma / mul / add per element, the same tables,
 * round-to-nearest-even), so the results are bit-identical to or_gate(..., ORACLE_FFT,
 * ...) -- tested.  The bootstrapping-key row of step i is shared by the lanes (broadcast)
 * and the transforms run on VL-wide vectors.  It exists so the CPU baseline is not
 * handicapped by a scalar port. */
#include <immintrin.h>

#ifdef __AVX512F__
#define OR_LANES 8
typedef __m512d vd;
typedef __m256i vu; /* OR_LANES x u32 */
#define VSET1 _mm512_set1_pd
#define VFMA _mm512_fmadd_pd
#define VADD _mm512_add_pd
#define VSUB _mm512_sub_pd
#define VMUL _mm512_mul_pd
#define VNEG(x) _mm512_xor_pd((x), _mm512_set1_pd(-0.0))
#define VCVT_I32 _mm512_cvtepi32_pd
#define ULOAD(p) _mm256_loadu_si256((const __m256i*)(p))
#define USTORE(p, x) _mm256_storeu_si256((__m256i*)(p), (x))
#define UADD _mm256_add_epi32
#define USUB _mm256_sub_epi32
#define UAND _mm256_and_si256
#define USET1 _mm256_set1_epi32
#define USRL _mm256_srl_epi32
/* llrint(r) mod 2^32 per lane: round to nearest even, exact int64, low word */
static inline vu low32_rint(vd r)
{
    return _mm512_cvtepi64_epi32(
        _mm512_cvtpd_epi64(_mm512_roundscale_pd(r, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC)));
}
#else
#define OR_LANES 4
typedef __m256d vd;
typedef __m128i vu;
#define VSET1 _mm256_set1_pd
#define VFMA _mm256_fmadd_pd
#define VADD _mm256_add_pd
#define VSUB _mm256_sub_pd
#define VMUL _mm256_mul_pd
#define VNEG(x) _mm256_xor_pd((x), _mm256_set1_pd(-0.0))
#define VCVT_I32 _mm256_cvtepi32_pd
#define ULOAD(p) _mm_loadu_si128((const __m128i*)(p))
#define USTORE(p, x) _mm_storeu_si128((__m128i*)(p), (x))
#define UADD _mm_add_epi32
#define USUB _mm_sub_epi32
#define UAND _mm_and_si128
#define USET1 _mm_set1_epi32
#define USRL _mm_srl_epi32
static inline vu low32_rint(vd x)
{
    /* round to nearest even; |r| < 2^51: low word of r + 1.5 * 2^52, else lane by lane */
    const vd r = _mm256_round_pd(x, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
    const vd ab = _mm256_andnot_pd(_mm256_set1_pd(-0.0), r);
    if (_mm256_movemask_pd(_mm256_cmp_pd(ab, _mm256_set1_pd(2251799813685248.0), _CMP_GE_OQ)) == 0) {
        const __m256i bits = _mm256_castpd_si256(_mm256_add_pd(r, _mm256_set1_pd(6755399441055744.0)));
        return _mm256_castsi256_si128(
            _mm256_permutevar8x32_epi32(bits, _mm256_setr_epi32(0, 2, 4, 6, 0, 2, 4, 6)));
    }
    double d[4];
    _mm256_storeu_pd(d, r);
    return _mm_setr_epi32((int)(uint32_t)(uint64_t)(int64_t)d[0], (int)(uint32_t)(uint64_t)(int64_t)d[1],
                          (int)(uint32_t)(uint64_t)(int64_t)d[2], (int)(uint32_t)(uint64_t)(int64_t)d[3]);
}
#endif

static inline void vbf_ct(vd* ur, vd* ui, vd* vr, vd* vi, vd c, vd nc, vd t, int rot)
{
    vd xr = *vr, xi = *vi;
    if (rot == 1) {
        const vd tmp = xr;
        xr = VNEG(xi);
        xi = tmp;
    } else if (rot == 3) {
        const vd tmp = xr;
        xr = xi;
        xi = VNEG(tmp);
    }
    const vd sr = VFMA(VNEG(xi), t, xr), si = VFMA(xr, t, xi);
    const vd a = *ur, b = *ui;
    *ur = VFMA(c, sr, a);
    *ui = VFMA(c, si, b);
    *vr = VFMA(nc, sr, a);
    *vi = VFMA(nc, si, b);
}

/* cmul: re = fma(x.re, w.re, -(x.im * w.im)), im = fma(x.re, w.im, x.im * w.re) */
static inline void vcmul(vd xr, vd xi, vd wr, vd wi, vd* rr, vd* ri)
{
    *rr = VFMA(xr, wr, VNEG(VMUL(xi, wi)));
    *ri = VFMA(xr, wi, VMUL(xi, wr));
}

static void vfwd_soa(const fft2_tab* T, vd* zr, vd* zi)
{
    const uint32_t M = OR_M;
    for (uint32_t s = 0; s < 9; s++) {
        const uint32_t h = M >> (s + 1);
        for (uint32_t b = 0; b < (1u << s); b++) {
            const int sib = (s % 3 != 0) && (b & 1);
            const uint32_t v = (1u << s) + b - (sib ? 1 : 0);
            const vd c = VSET1(T->fc[v]), nc = VSET1(-T->fc[v]), t = VSET1(T->ft[v]);
            const uint32_t o = 2 * h * b;
            for (uint32_t j = 0; j < h; j++)
                vbf_ct(&zr[o + j], &zi[o + j], &zr[o + j + h], &zi[o + j + h], c, nc, t, sib ? 1 : 0);
        }
    }
}

static void vinv_soa(const fft2_tab* T, vd* zr, vd* zi)
{
    const uint32_t M = OR_M;
    for (uint32_t h = 1; h < M; h <<= 1) {
        const uint32_t step = (M / 2) / h;
        for (uint32_t o = 0; o < M; o += 2 * h)
            for (uint32_t j = 0; j < h; j++) {
                const uint32_t e = j * step;
                vd *ur = &zr[o + j], *ui = &zi[o + j], *vr = &zr[o + j + h], *vi = &zi[o + j + h];
                if (h <= 4 && e == 0) { /* bf_1 */
                    const vd a = *ur, b = *ui, c = *vr, d = *vi;
                    *ur = VADD(a, c);
                    *ui = VADD(b, d);
                    *vr = VSUB(a, c);
                    *vi = VSUB(b, d);
                } else if (h <= 4 && e == M / 4) { /* bf_mi: -i v = (vi, -vr) */
                    const vd a = *ur, b = *ui, c = *vi, d = VNEG(*vr);
                    *ur = VADD(a, c);
                    *ui = VADD(b, d);
                    *vr = VSUB(a, c);
                    *vi = VSUB(b, d);
                } else if (h == 8 || h == 64) { /* bf_std with conj(W[e]) */
                    vd tr, ti;
                    vcmul(*vr, *vi, VSET1(T->W[e][0]), VSET1(-T->W[e][1]), &tr, &ti);
                    const vd a = *ur, b = *ui;
                    *ur = VADD(a, tr);
                    *ui = VADD(b, ti);
                    *vr = VSUB(a, tr);
                    *vi = VSUB(b, ti);
                } else {
                    const uint32_t e0 = e % (M / 4);
                    vbf_ct(ur, ui, vr, vi, VSET1(T->ic[e0]), VSET1(-T->ic[e0]), VSET1(-T->it[e0]),
                           e >= M / 4 ? 3 : 0);
                }
            }
    }
}

typedef struct {
    vd Fr[OR_M], Fi[OR_M];
    vd Ar[2][OR_M], Ai[2][OR_M];
    uint32_t tmp[2][OR_N][OR_LANES]; /* (X^a - 1) ACC, lane-interleaved */
    uint32_t acc[2][OR_N][OR_LANES]; /* ACC, lane-interleaved */
} simd_ws;

/* FFT-mode blind rotation + extraction of `lanes` (<= OR_LANES) combined LWE samples */
static void blind_rotate_extract_lanes(const or_keyset* ks, const uint32_t* const* lwe, int lanes,
                                       uint32_t mu, simd_ws* W, uint32_t* const* out_N)
{
    const or_params* p = &ks->p;
    const uint32_t n = p->n, N = p->N, M = N / 2, rows = (p->k + 1) * p->l;
    const fft2_tab* tab = get_tab(N);
    const uint32_t doff = decomp_offset(p);
    const uint32_t dmask = (1u << p->bgbit) - 1;
    const int32_t dhalf = 1 << (p->bgbit - 1);
    memset(W->acc, 0, sizeof(W->acc));
    for (int L = 0; L < lanes; L++) { /* ACC = (0, X^{-bbar} mu sum X^j) */
        const uint32_t e = (2 * N - or_mod_switch(lwe[L][n], N)) % (2 * N);
        for (uint32_t j = 0; j < N; j++) {
            const uint32_t idx = (j - e) & (2 * N - 1);
            W->acc[1][j][L] = idx < N ? mu : 0u - mu;
        }
    }
    for (uint32_t i = 0; i < n; i++) {
        uint32_t a[OR_LANES];
        int any = 0;
        int32_t lv[OR_LANES];
        for (int L = 0; L < OR_LANES; L++) {
            a[L] = L < lanes ? or_mod_switch(lwe[L][i], N) : 0;
            any |= a[L] != 0;
            lv[L] = a[L] ? -1 : 0; /* lanes whose external product is added (or_blind_rotate_acc skips a = 0) */
        }
        if (!any)
            continue;
        const vu live = ULOAD(lv);
        for (int L = 0; L < OR_LANES; L++)
            for (uint32_t c = 0; c < 2; c++)
                for (uint32_t j = 0; j < N; j++) { /* (X^a P)_j - P_j, a in [0, 2N) */
                    const uint32_t idx = (j - a[L]) & (2 * N - 1);
                    const uint32_t pv = W->acc[c][idx & (N - 1)][L];
                    W->tmp[c][j][L] = (idx < N ? pv : 0u - pv) - W->acc[c][j][L];
                }
        memset(W->Ar, 0, sizeof(W->Ar));
        memset(W->Ai, 0, sizeof(W->Ai));
        for (uint32_t c = 0; c < 2; c++)
            for (uint32_t q = 0; q < p->l; q++) {
                /* or_decompose lane-wise: ((x + off) >> shift) & mask - half, then exact (double) */
                const vu voff = USET1((int)doff), vmask = USET1((int)dmask), vhalf = USET1(dhalf);
                const __m128i vsh = _mm_cvtsi32_si128((int)(32 - (q + 1) * p->bgbit));
                for (uint32_t j = 0; j < M; j++) {
                    const vu d0 = USUB(UAND(USRL(UADD(ULOAD(W->tmp[c][j]), voff), vsh), vmask), vhalf);
                    const vu d1 = USUB(UAND(USRL(UADD(ULOAD(W->tmp[c][j + M]), voff), vsh), vmask), vhalf);
                    W->Fr[j] = VCVT_I32(d0);
                    W->Fi[j] = VCVT_I32(d1);
                }
                vfwd_soa(tab, W->Fr, W->Fi);
                const uint32_t r = c * p->l + q;
                for (uint32_t comp = 0; comp < 2; comp++) {
                    const double* Br = ks->bk_fft_soa + (((size_t)i * rows + r) * 2 + comp) * N;
                    const double* Bi = Br + M;
                    vd* ar = W->Ar[comp];
                    vd* ai = W->Ai[comp];
                    for (uint32_t f = 0; f < M; f++) {
                        const vd br = VSET1(Br[f]), bi = VSET1(Bi[f]);
                        vd re = VFMA(W->Fr[f], br, ar[f]);
                        re = VFMA(VNEG(W->Fi[f]), bi, re);
                        vd im = VFMA(W->Fr[f], bi, ai[f]);
                        im = VFMA(W->Fi[f], br, im);
                        ar[f] = re;
                        ai[f] = im;
                    }
                }
            }
        for (uint32_t comp = 0; comp < 2; comp++) {
            vd* zr = W->Ar[comp];
            vd* zi = W->Ai[comp];
            vinv_soa(tab, zr, zi);
            for (uint32_t j = 0; j < M; j++) { /* untwist, round, ACC += (a != 0 lanes) */
                vd wr, wi;
                vcmul(zr[j], zi[j], VSET1(tab->TW[j][0]), VSET1(-tab->TW[j][1]), &wr, &wi);
                uint32_t* a0 = W->acc[comp][j];
                uint32_t* a1 = W->acc[comp][j + M];
                USTORE(a0, UADD(ULOAD(a0), UAND(low32_rint(wr), live)));
                USTORE(a1, UADD(ULOAD(a1), UAND(low32_rint(wi), live)));
            }
        }
    }
    for (int L = 0; L < lanes; L++) { /* sample extraction at index 0 */
        uint32_t* o = out_N[L];
        o[0] = W->acc[0][0][L];
        for (uint32_t j = 1; j < N; j++)
            o[j] = 0u - W->acc[0][N - j][L];
        o[N] = W->acc[1][0][L];
    }
}

typedef struct {
    const or_keyset* ks;
    int kind;
    const uint32_t *a, *b;
    uint32_t* out;
    uint64_t lo, hi;
    int rc;
} simd_job;

static void* simd_worker(void* arg)
{
    simd_job* jb = (simd_job*)arg;
    const or_keyset* ks = jb->ks;
    const uint32_t n = ks->p.n, N = ks->p.N;
    const size_t w = n + 1;
    simd_ws* W = (simd_ws*)aligned_alloc(64, (sizeof(simd_ws) + 63) / 64 * 64);
    uint32_t* comb = (uint32_t*)malloc(sizeof(uint32_t) * w * OR_LANES);
    uint32_t* ext = (uint32_t*)malloc(sizeof(uint32_t) * (N + 1) * OR_LANES);
    for (uint64_t g0 = jb->lo; g0 < jb->hi; g0 += OR_LANES) {
        const int lanes = (int)(jb->hi - g0 < OR_LANES ? jb->hi - g0 : OR_LANES);
        const uint32_t* lw[OR_LANES];
        uint32_t* eo[OR_LANES];
        for (int L = 0; L < OR_LANES; L++) {
            lw[L] = comb + (size_t)L * w;
            eo[L] = ext + (size_t)L * (N + 1);
        }
        for (int L = 0; L < lanes; L++) {
            const uint32_t* A = jb->a + (g0 + L) * w;
            const uint32_t* B = jb->b + (g0 + L) * w;
            uint32_t* cb = comb + (size_t)L * w;
            switch (jb->kind) {
            case OR_GATE_AND: lin2(n, 0xE0000000u, 1, A, 1, B, cb); break;
            case OR_GATE_OR: lin2(n, 0x20000000u, 1, A, 1, B, cb); break;
            case OR_GATE_XOR: lin2(n, 0x40000000u, 2, A, 2, B, cb); break;
            case OR_GATE_XNOR: lin2(n, 0xC0000000u, -2, A, -2, B, cb); break;
            case OR_GATE_NAND: lin2(n, 0x20000000u, -1, A, -1, B, cb); break;
            case OR_GATE_NOR: lin2(n, 0xE0000000u, -1, A, -1, B, cb); break;
            default: jb->rc = -1; goto out;
            }
        }
        blind_rotate_extract_lanes(ks, lw, lanes, 0x20000000u, W, eo);
        for (int L = 0; L < lanes; L++)
            or_keyswitch(ks, eo[L], jb->out + (g0 + L) * w);
    }
out:
    free(W);
    free(comb);
    free(ext);
    return NULL;
}

int or_simd_lanes(void) { return OR_LANES; }

int or_gate_batch_simd(const or_keyset* ks, int kind, const uint32_t* a, const uint32_t* b,
                       uint32_t* out, uint64_t count, int threads)
{
    if (ks->p.N != OR_N)
        return -1;
    if (threads < 1)
        threads = 1;
    const uint64_t groups = (count + OR_LANES - 1) / OR_LANES;
    if ((uint64_t)threads > groups)
        threads = groups ? (int)groups : 1;
    simd_job* jobs = (simd_job*)calloc(threads, sizeof(simd_job));
    pthread_t* tid = (pthread_t*)calloc(threads, sizeof(pthread_t));
    const uint64_t chunk = (groups + threads - 1) / threads * OR_LANES; /* whole lane groups */
    for (int t = 0; t < threads; t++) {
        jobs[t].ks = ks;
        jobs[t].kind = kind;
        jobs[t].a = a;
        jobs[t].b = b;
        jobs[t].out = out;
        jobs[t].lo = (uint64_t)t * chunk < count ? (uint64_t)t * chunk : count;
        jobs[t].hi = jobs[t].lo + chunk < count ? jobs[t].lo + chunk : count;
    }
    for (int t = 1; t < threads; t++)
        pthread_create(&tid[t], NULL, simd_worker, &jobs[t]);
    simd_worker(&jobs[0]);
    int rc = jobs[0].rc;
    for (int t = 1; t < threads; t++) {
        pthread_join(tid[t], NULL);
        if (jobs[t].rc)
            rc = jobs[t].rc;
    }
    free(jobs);
    free(tid);
    return rc;
}

/* A heterogeneous gate list (one level of a gate program) lane-batched like
 * or_gate_batch_simd: every item's blind rotation(s) -- one per gate, two for a MUX --
 * are gathered, rotated VL at a time, then key-switched per item exactly as or_gate does
 * (bit-identical to or_gate_list(..., ORACLE_FFT, ...)). */
typedef struct {
    const or_keyset* ks;
    const or_gate_item* items;
    uint64_t lo, hi;
    int rc;
} list_simd_job;

static void* list_simd_worker(void* arg)
{
    list_simd_job* jb = (list_simd_job*)arg;
    const or_keyset* ks = jb->ks;
    const uint32_t n = ks->p.n, N = ks->p.N;
    const size_t w = n + 1;
    const uint64_t cnt = jb->hi - jb->lo;
    uint64_t nbr = 0;
    for (uint64_t g = jb->lo; g < jb->hi; g++)
        nbr += jb->items[g].kind == OR_GATE_MUX ? 2 : 1;
    uint32_t* comb = (uint32_t*)malloc(sizeof(uint32_t) * w * (nbr + OR_LANES));
    uint32_t* ext = (uint32_t*)malloc(sizeof(uint32_t) * (N + 1) * (nbr + OR_LANES));
    uint64_t* first = (uint64_t*)malloc(sizeof(uint64_t) * (cnt + 1));
    simd_ws* W = (simd_ws*)aligned_alloc(64, (sizeof(simd_ws) + 63) / 64 * 64);
    uint64_t k = 0;
    for (uint64_t g = jb->lo; g < jb->hi; g++) { /* linear forms (or_gate) */
        const or_gate_item* it = &jb->items[g];
        uint32_t* cb = comb + k * w;
        first[g - jb->lo] = k;
        switch (it->kind) {
        case OR_GATE_AND: lin2(n, 0xE0000000u, 1, it->a, 1, it->b, cb); break;
        case OR_GATE_OR: lin2(n, 0x20000000u, 1, it->a, 1, it->b, cb); break;
        case OR_GATE_XOR: lin2(n, 0x40000000u, 2, it->a, 2, it->b, cb); break;
        case OR_GATE_XNOR: lin2(n, 0xC0000000u, -2, it->a, -2, it->b, cb); break;
        case OR_GATE_NAND: lin2(n, 0x20000000u, -1, it->a, -1, it->b, cb); break;
        case OR_GATE_NOR: lin2(n, 0xE0000000u, -1, it->a, -1, it->b, cb); break;
        case OR_GATE_ANDNY: lin2(n, 0xE0000000u, -1, it->a, 1, it->b, cb); break;
        case OR_GATE_ORNY: lin2(n, 0x20000000u, -1, it->a, 1, it->b, cb); break;
        case OR_GATE_MAJ:
            lin2(n, 0u, 1, it->a, 1, it->b, cb);
            for (uint32_t q = 0; q <= n; q++)
                cb[q] += it->c[q];
            break;
        case OR_GATE_XOR3:
            lin2(n, 0u, -2, it->a, -2, it->b, cb);
            for (uint32_t q = 0; q <= n; q++)
                cb[q] += (uint32_t)-2 * it->c[q];
            break;
        case OR_GATE_MUX:
            lin2(n, 0xE0000000u, 1, it->a, 1, it->b, cb);
            lin2(n, 0xE0000000u, -1, it->a, 1, it->c, cb + w);
            k++;
            break;
        default: jb->rc = -1; goto out;
        }
        k++;
    }
    for (uint64_t g0 = 0; g0 < nbr; g0 += OR_LANES) { /* blind rotations, VL at a time */
        const int lanes = (int)(nbr - g0 < OR_LANES ? nbr - g0 : OR_LANES);
        const uint32_t* lw[OR_LANES];
        uint32_t* eo[OR_LANES];
        for (int L = 0; L < OR_LANES; L++) {
            lw[L] = comb + (g0 + L) * w;
            eo[L] = ext + (g0 + L) * (N + 1);
        }
        blind_rotate_extract_lanes(ks, lw, lanes, 0x20000000u, W, eo);
    }
    for (uint64_t g = jb->lo; g < jb->hi; g++) { /* key switches (or_gate) */
        const or_gate_item* it = &jb->items[g];
        uint32_t* e = ext + first[g - jb->lo] * (N + 1);
        if (it->kind == OR_GATE_MUX) {
            const uint32_t* e2 = e + (N + 1);
            for (uint32_t q = 0; q <= N; q++)
                e[q] += e2[q];
            e[N] += 0x20000000u;
        }
        or_keyswitch(ks, e, it->out);
    }
out:
    free(comb);
    free(ext);
    free(first);
    free(W);
    return NULL;
}

int or_gate_list_simd(const or_keyset* ks, const or_gate_item* items, uint64_t count, int threads)
{
    if (ks->p.N != OR_N)
        return -1;
    if (threads < 1)
        threads = 1;
    if ((uint64_t)threads > count)
        threads = count ? (int)count : 1;
    list_simd_job* jobs = (list_simd_job*)calloc(threads, sizeof(list_simd_job));
    pthread_t* tid = (pthread_t*)calloc(threads, sizeof(pthread_t));
    const uint64_t chunk = (count + threads - 1) / threads;
    for (int t = 0; t < threads; t++) {
        jobs[t].ks = ks;
        jobs[t].items = items;
        jobs[t].lo = (uint64_t)t * chunk < count ? (uint64_t)t * chunk : count;
        jobs[t].hi = jobs[t].lo + chunk < count ? jobs[t].lo + chunk : count;
    }
    for (int t = 1; t < threads; t++)
        pthread_create(&tid[t], NULL, list_simd_worker, &jobs[t]);
    list_simd_worker(&jobs[0]);
    int rc = jobs[0].rc;
    for (int t = 1; t < threads; t++) {
        pthread_join(tid[t], NULL);
        if (jobs[t].rc)
            rc = jobs[t].rc;
    }
    free(jobs);
    free(tid);
    return rc;
}
