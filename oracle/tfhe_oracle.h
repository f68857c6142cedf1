/*
 * tfhe_oracle.h -- CPU ORACLE for the LocPIR gate-bootstrapping hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or as the timed CPU baseline.  The product path
 * (paper_2407_19871_b200/) never links, loads or calls anything here.
 *
 * What it restates, and how it is pinned:
 *  - LWE layer (torus words, NoiseSampler = mt19937_64 + libstdc++
 *    normal_distribution, keygen, encrypt, phase, decrypt, linear ops) follows
 *    /root/reference/proj/include/locpir/torus.hpp:19-222.  PINNED bit-exactly
 *    against golden vectors produced by the reference itself compiled here
 *    (oracle/ref_driver.cpp -> tests/golden/ref_vectors.json).
 *  - Gate linear forms and MUX structure follow gate_engine.hpp:196-269;
 *    counting follows gate_engine.hpp:31-77; circuits follow
 *    circuits.hpp:187-324.  Decrypted behaviour PINNED against the reference's
 *    own tests (truth tables, comparator order, loc_pir retrieval, gate counts)
 *    and against reference-generated goldens.
 *  - The real gate bootstrap (blind rotation, TRGSW external product,
 *    negacyclic FFT, sample extraction, key switching) is NOT in the reference:
 *    the reference uses a secret-key refresh stand-in (gate_engine.hpp:117-123)
 *    and the paper delegates to "TFHE library version 1.1",
 *    a third-party dependency that is absent from /root/reference, not
 *    vendored and not pinned.  Its published algorithm is restated here in
 *    plain C.  No ciphertext-level golden vector of TFHE 1.1 exists in the
 *    reference, so the bootstrap INTERNALS are "parity unpinned" against
 *    TFHE 1.1; they are anchored on (a) the reference's gate-level and
 *    circuit-level pins above and (b) internal consistency: the FFT-mode
 *    external product is checked against an exact mod-2^32 schoolbook product.
 *
 * Two polynomial back ends: ORACLE_EXACT (schoolbook, the ground truth) and
 * ORACLE_FFT (FP64 negacyclic FFT whose arithmetic -- radix-2 DIF forward,
 * radix-2 DIT inverse, fixed fma patterns, the twiddle tables below -- is the
 * contract the B200 kernels reproduce bit-for-bit).
 */
#ifndef LOCPIR_TFHE_ORACLE_H
#define LOCPIR_TFHE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- mt19937_64 and the reference NoiseSampler (torus.hpp:119-138) ---- */
typedef struct {
    uint64_t mt[312];
    int mti;
} or_mt64;

void or_mt64_seed(or_mt64* g, uint64_t seed);
uint64_t or_mt64_next(or_mt64* g);

typedef struct {
    or_mt64 rng;
    double sigma;
} or_sampler;

void or_sampler_init(or_sampler* s, uint64_t seed, double sigma);
uint32_t or_sampler_uniform(or_sampler* s);
uint32_t or_sampler_gaussian(or_sampler* s);
double or_gaussian_double(or_sampler* s); /* raw N(0, sigma) draw */
uint32_t or_torus_from_double(double x);  /* torus.hpp:38-43 */
uint64_t or_child_seed(uint64_t seed, uint64_t lane); /* gate_engine.hpp:601-607 */

/* ---- LWE layer (torus.hpp) ----
 * A sample is n+1 u32 words, mask first, body last (wire order, torus.hpp:226-237). */
void or_keygen(uint32_t n, uint64_t seed, uint8_t* bits_out);
void or_encrypt_torus(uint32_t mu, const uint8_t* key, uint32_t n, or_sampler* s,
                      uint32_t* out);
void or_encrypt_bit(int bit, const uint8_t* key, uint32_t n, or_sampler* s, uint32_t* out);
uint32_t or_phase(const uint32_t* ct, const uint8_t* key, uint32_t n);
int or_decrypt_bit(const uint32_t* ct, const uint8_t* key, uint32_t n);
/* The reference refresh stand-in (gate_engine.hpp:117-123), kept to pin the LWE layer. */
void or_bootstrap_standin(const uint32_t* ct, const uint8_t* key, uint32_t n, or_sampler* s,
                          uint32_t* out);

/* ---- TFHE parameters (BASELINE.json configs[0], [1]) ---- */
typedef struct {
    uint32_t n, N, k, l, bgbit, t, basebit;
    double alpha_in, alpha_bk;
} or_params;

void or_params_default(int level, or_params* p); /* level 80 or 128 */

typedef struct {
    or_params p;
    uint8_t* lwe_key;   /* n bits */
    uint8_t* trlwe_key; /* N bits */
    uint32_t* bk;       /* torus form [n][(k+1)l][k+1][N] */
    uint32_t* ksk;      /* [N][t][base-1][n+1] */
    double* bk_fft;     /* [n][(k+1)l][k+1][N/2][2] (re,im), slot order, scaled by 1/(N/2) */
    double* bk_fft_soa; /* same values, [..][k+1][re[N/2], im[N/2]] (vectorisable MAC) */
} or_keyset;

/* Deterministic key set from one seed. */
int or_keyset_generate(or_keyset* ks, const or_params* p, uint64_t seed);
void or_keyset_free(or_keyset* ks);
size_t or_bk_words(const or_params* p);
size_t or_ksk_words(const or_params* p);

/* ---- negacyclic transform (N real -> N/2 complex), N = 1024 only ---- */
/* the transform's tables (tfhe_oracle.c): forward twiddle base (cos, tan) per tree node
 * [M], W^e [M/2][2], inverse base (cos, tan) [M/4], factored twist [M][2] */
void or_fft2_make_tables(double* fc, double* ft, double* W, double* ic, double* it, double* TW);
void or_fft_tables(uint32_t N, double* W /*[N/4][2]*/, double* TW /*[N/2][2]*/,
                   double* UT /*[N/2][2]*/);
void or_fft_forward_i32(uint32_t N, const int32_t* in, double* out /*[N/2][2]*/);
/* inverse transform; rounds each coefficient to the nearest integer mod 2^32 and
 * ADDS it into acc[N]. in[] is destroyed. */
void or_fft_inverse_add(uint32_t N, double* in, uint32_t* acc);
/* max |w - rint(w)| over every inverse output since the last reset (FFT rounding margin) */
double or_fft_margin(int reset);
/* exact negacyclic product mod 2^32: acc += d * b */
void or_polymul_exact_add(uint32_t N, const int32_t* d, const uint32_t* b, uint32_t* acc);

enum { ORACLE_EXACT = 0, ORACLE_FFT = 1 };

/* Gadget decomposition of one polynomial, digit p in [0, l). */
void or_decompose(const or_params* p, const uint32_t* x, uint32_t level, int32_t* digits);

/* mod switch one torus word to [0, 2N) */
uint32_t or_mod_switch(uint32_t x, uint32_t N);

/* Blind rotation + sample extraction of an n-dim LWE (already combined).
 * Output: N-dim LWE (N+1 words).  mu = test-vector value. */
int or_blind_rotate_extract(const or_keyset* ks, const uint32_t* lwe_in, uint32_t mu,
                            int mode, uint32_t* out_N);
/* Same but stop after `steps` CMux iterations and return the raw accumulator
 * (2N words, A then B) -- used for stage-wise KATs. */
int or_blind_rotate_acc(const or_keyset* ks, const uint32_t* lwe_in, uint32_t mu, int mode,
                        uint32_t steps, uint32_t* acc_out);
/* external product of a TRLWE (2N words) with BK_i; mode exact/FFT; out = 2N words */
int or_external_product(const or_keyset* ks, uint32_t i, const uint32_t* trlwe, int mode,
                        uint32_t* out);
/* N-dim -> n-dim key switch */
void or_keyswitch(const or_keyset* ks, const uint32_t* in_N, uint32_t* out_n);

/* ---- gates (gate_engine.hpp:196-269 forms, TFHE bootstrap) ---- */
enum {
    OR_GATE_AND = 0,
    OR_GATE_OR = 1,
    OR_GATE_XOR = 2,
    OR_GATE_XNOR = 3,
    OR_GATE_NAND = 4,
    OR_GATE_MUX = 5,
    OR_GATE_NOT = 6,
    OR_GATE_NOR = 7,
    OR_GATE_ANDNY = 10, /* AND(NOT a, b): flagged constant-folding mode */
    OR_GATE_ORNY = 11,  /* OR(NOT a, b) */
    OR_GATE_MAJ = 12,   /* MAJ(a, b, c) = BS(a + b + c): flagged majority-comparator mode */
    OR_GATE_XOR3 = 13   /* a ^ b ^ c = BS(-2 (a + b + c)): flagged ternary XOR trees */
};
/* out = gate(a, b[, c]) ; for MUX: out = a ? b : c.  n-dim in/out. */
int or_gate(const or_keyset* ks, int kind, const uint32_t* a, const uint32_t* b,
            const uint32_t* c, int mode, uint32_t* out);
/* Batched gates on `threads` host threads (static block partition as
 * parallel.hpp:15-52).  a,b,out are [count][n+1]. */
int or_gate_batch(const or_keyset* ks, int kind, const uint32_t* a, const uint32_t* b,
                  uint32_t* out, uint64_t count, int mode, int threads);
/* The same FFT-mode 2-input gates, or_simd_lanes() ciphertexts per SIMD lane group (8 with
 * AVX-512, 4 with AVX2; bit-identical to or_gate_batch(..., ORACLE_FFT, ...)); the CPU
 * baseline's fast path. */
int or_simd_lanes(void);
int or_gate_batch_simd(const or_keyset* ks, int kind, const uint32_t* a, const uint32_t* b,
                       uint32_t* out, uint64_t count, int threads);

/* Counter-based client encryption (paper_2407_19871_b200/csrc/cbrng.h):
 * sample j = (mask philox words, body = <a, key> + mus[j] + noise) with stream index
 * first_index + j.  Also exported: the Philox block and the Gaussian pieces for pins. */
void or_cb_encrypt(const uint8_t* key, uint32_t n, uint64_t seed, uint32_t first_index,
                   const uint32_t* mus, uint64_t count, double alpha, uint32_t* out);
void or_cb_philox(const uint32_t ctr[4], uint64_t seed, uint32_t out[4]);
double or_cb_log(double u);
double or_cb_cos2pi(double x);
uint32_t or_cb_noise(uint64_t seed, uint32_t index, double alpha);

/* Heterogeneous gate list on `threads` host threads (static block partition as
 * parallel.hpp:15-52): one level of a gate program. */
typedef struct {
    int kind;
    const uint32_t *a, *b, *c;
    uint32_t* out;
} or_gate_item;
int or_gate_list(const or_keyset* ks, const or_gate_item* items, uint64_t count, int mode,
                 int threads);
/* The same list in FFT mode, blind rotations lane-batched (bit-identical; CPU baseline). */
int or_gate_list_simd(const or_keyset* ks, const or_gate_item* items, uint64_t count,
                      int threads);

#ifdef __cplusplus
}
#endif
#endif
