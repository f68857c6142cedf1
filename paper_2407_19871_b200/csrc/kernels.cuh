// kernels.cuh -- B200 (sm_100a) kernels of the gate-bootstrapping hot path.
//
//   K0 k_bk_to_freq    : torus-form BK -> FP64 frequency domain (once per GPU)
//   K1 k_blind_rotate  : gate prologue (linear combination + mod switch), blind
//                        rotation (n CMux external products against BK_i),
//                        sample extraction  -> N-dim LWE
//   K2 k_keyswitch     : (sum of <= 2 N-dim LWE + offset) -> n-dim LWE, streaming
//                        the KSK; also realises the MUX combine (TFHE bootsMUX)
//   K3 k_linear        : free gates (NOT, COPY, CONST)
//
// The algorithm is SURVEY.md §8(a') (TFHE gate bootstrapping), restated with the
// same arithmetic as oracle/tfhe_oracle.c; the linear gate forms are the
// reference's (gate_engine.hpp:196-269).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cassert>

#include "fft.cuh"
#include "cbrng.h"

namespace lpb {

constexpr uint32_t SLOT_NONE = 0xFFFFFFFFu;

// One blind rotation: combined = off + c0 * in0 + c1 * in1 + c2 * in2 (n-dim; in1 / in2
// optional), output N-dim.  The third input serves the 3-input majority gate.
struct BrItem {
    uint32_t in0, in1;
    int32_t c0, c1;
    uint32_t off;
    uint32_t out;  // N-dim scratch slot
    uint32_t in2;
    int32_t c2;
};

// One key switch: combined = in0 + in1 (N-dim, in1 optional) + (0, off) -> n-dim slot.
struct KsItem {
    uint32_t in0, in1;
    uint32_t off;
    uint32_t out;
};

// One free gate.
struct LinItem {
    uint32_t kind;  // 0 NOT, 1 COPY, 2 CONST
    uint32_t in0;   // slot (NOT/COPY) or constant word (CONST)
    uint32_t out;
    uint32_t pad;
};

struct DevParams {
    uint32_t n, N, l, bgbit, t, basebit;
    uint32_t n_stride;  // padded n+1
    uint32_t N_stride;  // padded N+1
    uint64_t pool_slots, scratch_slots;  // current pool sizes (bounds for LPB_CHECKS)
    // zero-copy inputs of one gate_batch_host call: packed [count][n+1] rows in pinned,
    // device-mapped host memory, addressed by the slots SLOT_EXT_A / SLOT_EXT_B | row
    const uint32_t* ext_a;
    const uint32_t* ext_b;
    uint32_t ext_rows;
};
constexpr uint32_t SLOT_EXT_A = 0x80000000u, SLOT_EXT_B = 0xC0000000u, SLOT_EXT_ROW = 0x3FFFFFFFu;


// ---- self-check build (compute-sanitizer is closed on the GPU pool):
//   LPB_CHECKS=1  device asserts on every pool / scratch / table index a kernel forms
//   LPB_JITTER=1  a pseudo-random __nanosleep before every barrier and warp sync, so a
//                 missing or misplaced barrier shows up as a result that changes from run
//                 to run (tools/selfcheck.sh compares digests across runs and poisons)
#ifndef LPB_CHECKS
#define LPB_CHECKS 0
#endif
#ifndef LPB_JITTER
#define LPB_JITTER 0
#endif
#if LPB_CHECKS
#define LPB_ASSERT(x) assert(x)
#else
#define LPB_ASSERT(x) ((void)0)
#endif
// An input LWE row: a pool slot, or (gate_batch_host's zero-copy path) a row of the
// caller's pinned host buffer read over PCIe by the blind rotation's prologue.
__device__ __forceinline__ const uint32_t* lwe_row(const DevParams& dp, const uint32_t* pool_n,
                                                   uint32_t slot)
{
    if (slot >= SLOT_EXT_A) {
        LPB_ASSERT((slot & SLOT_EXT_ROW) < dp.ext_rows);
        return ((slot & 0x40000000u) ? dp.ext_b : dp.ext_a) + (size_t)(slot & SLOT_EXT_ROW) * (dp.n + 1);
    }
    LPB_ASSERT(slot < dp.pool_slots);
    return pool_n + (size_t)slot * dp.n_stride;
}

__constant__ uint32_t c_poison;  // LOCPIR_B200_POISON (checked build: shared memory poison)

__global__ void k_fill(uint32_t* __restrict__ p, size_t words, uint32_t v)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < words;
         i += (size_t)gridDim.x * blockDim.x)
        p[i] = v;
}

// checked build: fill this CTA's shared memory with the poison word before use
__device__ __forceinline__ void lpb_poison_smem(void* base, size_t bytes)
{
#if LPB_CHECKS
    uint32_t* w = reinterpret_cast<uint32_t*>(base);
    for (size_t i = threadIdx.x; i < bytes / 4; i += blockDim.x)
        w[i] = c_poison;
    __syncthreads();
#else
    (void)base;
    (void)bytes;
#endif
}

__device__ __forceinline__ void lpb_jitter()
{
#if LPB_JITTER
    unsigned s = (unsigned)clock() * 2654435761u ^ (threadIdx.x * 0x9E3779B9u) ^ blockIdx.x;
    __nanosleep((s >> 20) & 511u);
#endif
}

// The transform's device tables (engine.cu make_tables; same values as the oracle's
// or_fft2_make_tables): per-thread forward / inverse twiddles [8][64] and the factored
// twist psi^j (the untwist is its conjugate).
struct FftTabs {
    const double2* fwd;
    const double2* inv;
    const double2* tw;
};
__constant__ double2 c_twq[8];  // psi^(64 q), q = 0..7: psi^(t + 64 q) = cmul(psi^t, psi^(64 q))

// untwist factor conj(psi^(t + 64 q)) from the thread's psi^t
__device__ __forceinline__ double2 untwist(double2 twt, int q) { return conj2(cmul(twt, c_twq[q])); }

// ---------------------------------------------------------------------------
// K0: BK torus polynomials -> frequency domain (scaled by 1/512, exact), layout
// [poly][q*64 + t] where the frequency slot is 8t + q (K1's per-thread loads coalesce).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(64) k_bk_to_freq(const uint32_t* __restrict__ bk,
                                                   double2* __restrict__ out, FftTabs tb)
{
    __shared__ __align__(16) double2 xbuf[2][XTILE];
    const int t = threadIdx.x;
    const size_t poly = blockIdx.x;
    const uint32_t* b = bk + poly * 1024;
    const FwdTw tw = load_fwd_tw(tb.fwd, t);
    double2 x[8];
#pragma unroll
    for (int q = 0; q < 8; q++) {
        const int j = t + 64 * q;
        x[q] = make_double2((double)(int32_t)b[j], (double)(int32_t)b[j + 512]);
    }
    auto bar = [] { __syncthreads(); };
    auto wbar = [] { __syncwarp(); };
    fft_forward(x, tw, xbuf[0], xbuf[1], t, bar, wbar);
    double2* o = out + poly * FFT_M;
#pragma unroll
    for (int q = 0; q < 8; q++)
        o[q * 64 + t] = make_double2(x[q].x * (1.0 / 512.0), x[q].y * (1.0 / 512.0));
}

// ---------------------------------------------------------------------------
// K1: blind rotation + sample extraction, one 64-thread CTA per ciphertext.
// ---------------------------------------------------------------------------
// Largest LWE dimension the device kernels are built for: K2 covers KS_THREADS x KS_COLS
// = 640 output columns (n+1 padded to 4), ctx_create rejects n > 636; abar arrays hold
// MAX_N + 1 entries.
constexpr int MAX_N = 639;
constexpr uint32_t MAX_CTX_N = 636;
#ifndef LAT_BK_SPREAD
#define LAT_BK_SPREAD 1  // K1l: BK loads issued between the forward passes
#endif
#ifndef LAT_BK_B0
#define LAT_BK_B0 2  // rows loaded before pass 0 / before pass 1 (cumulative) / rest before pass 2
#endif
#ifndef LAT_BK_B1
#define LAT_BK_B1 4
#endif
#ifndef BR_MIN_BLOCKS
#define BR_MIN_BLOCKS 4  // ciphertexts resident per SM (255 registers per thread)
#endif

__device__ __forceinline__ uint32_t rot_read(const uint32_t* p, uint32_t a, int j)
{
    // (X^a * P)_j for a in [0, 2N), N = 1024
    const uint32_t idx = (uint32_t)(j - (int)a) & 2047u;
    const uint32_t v = p[idx & 1023u];
    return idx < 1024u ? v : 0u - v;
}

// BK rows are streamed once per CTA per step: kept out of L1 and pinned in L2
// (evict_last).  A relaxed gpu-scope load may not be sunk below the transform's
// bar.sync by ptxas (a weak .nc load is, which turns the prefetch into a stall at the MAC).
__device__ __forceinline__ double2 ld_stream(const double2* p)
{
    double2 v;
    asm volatile(
        "{\n\t.reg .b64 pol;\n\t"
        "createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
        "ld.relaxed.gpu.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], pol;\n\t}"
        : "=d"(v.x), "=d"(v.y)
        : "l"(p));
    return v;
}

// Integer <-> double conversions on the FP64 pipe instead of the conversion unit (XU):
// digit_to_double(u) = u - HALF for a field value u < 2^20, exact: the bit pattern 2^52 + u
// minus (2^52 + HALF).  round_low32<SAFE>(w) = rint(w) mod 2^32 (ties to even, as
// __double2ll_rn): with |w| < 2^51 the sum w + 1.5 * 2^52 is rounded to an integer and its
// low word is rint(w) mod 2^32.  The external product bounds |w| by 2l N 2^(Bgbit-1) 2^31
// (+ the < 1/2 transform error): 2^49.6 at 128-bit, so SAFE; 2^52 at 80-bit, which keeps
// the conversion instruction.
__device__ __forceinline__ double digit_to_double(uint32_t u, uint32_t half)
{
    return __dsub_rn(__hiloint2double(0x43300000, (int)u), 4503599627370496.0 + (double)half);
}
template <bool SAFE>
__device__ __forceinline__ uint32_t round_low32(double w)
{
    if constexpr (SAFE)
        return (uint32_t)__double2loint(__dadd_rn(w, 6755399441055744.0));
    else
        return (uint32_t)__double2ll_rn(w);
}
template <int L, int BGBIT>
constexpr bool kMagicRound = (1ull << (BGBIT - 1)) * (2ull * L) * 1024ull < (1ull << 20);
static_assert(kMagicRound<3, 7>, "128-bit: |w| <= 6 * 1024 * 2^6 * 2^31 = 2^49.6 < 2^51");
static_assert(!kMagicRound<2, 10>, "80-bit: the bound 4 * 1024 * 2^9 * 2^31 = 2^52 is not < 2^51");

__device__ __forceinline__ void mac(double2& acc, double2 F, double2 B)
{
    double re = __fma_rn(F.x, B.x, acc.x);
    re = __fma_rn(-F.y, B.y, re);
    double im = __fma_rn(F.x, B.y, acc.y);
    im = __fma_rn(F.y, B.x, im);
    acc.x = re;
    acc.y = im;
}

// ERR = true (diagnostic instantiation only): also record max |w - rint(w)| over every
// inverse-transform output before rounding -- the FFT rounding margin (exact iff < 1/2).
template <int L, int BGBIT, bool ERR = false>
__global__ void __launch_bounds__(64, BR_MIN_BLOCKS)
    k_blind_rotate(DevParams dp, const BrItem* __restrict__ items,
                   const uint32_t* __restrict__ pool_n, uint32_t* __restrict__ pool_N,
                   const double2* __restrict__ bkf, FftTabs tb, uint32_t mu,
                   unsigned long long* err_out = nullptr)
{
    double emax = 0.0;
    __shared__ uint32_t acc[2][1024];
    // exchange tiles: [0],[1] cross-warp (alternating), [2] intra-warp
    __shared__ __align__(16) double2 xbuf[3][XTILE];
    __shared__ uint16_t abar[MAX_N + 1];

    const int t = threadIdx.x;
    const BrItem it = items[blockIdx.x];
    const uint32_t n = dp.n;
    LPB_ASSERT(it.out < dp.scratch_slots && n <= MAX_N);
#if LPB_CHECKS
    lpb_poison_smem(acc, sizeof(acc));
    lpb_poison_smem(xbuf, sizeof(xbuf));
    lpb_poison_smem(abar, sizeof(abar));
#endif

    // ---- prologue: gate linear form (gate_engine.hpp:196-269) + mod switch to [0, 2N)
    {
        const uint32_t* a0 = lwe_row(dp, pool_n, it.in0);
        const uint32_t* a1 = it.in1 != SLOT_NONE ? lwe_row(dp, pool_n, it.in1) : nullptr;
        const uint32_t* a2 = it.in2 != SLOT_NONE ? lwe_row(dp, pool_n, it.in2) : nullptr;
        for (uint32_t i = t; i <= n; i += 64) {
            uint32_t v = (uint32_t)it.c0 * a0[i];
            if (a1)
                v += (uint32_t)it.c1 * a1[i];
            if (a2)
                v += (uint32_t)it.c2 * a2[i];
            if (i == n)
                v += it.off;
            abar[i] = (uint16_t)((v + (1u << 20)) >> 21);  // round(v * 2N / 2^32), N = 1024
        }
    }
    __syncthreads();
    // ---- test vector: ACC = (0, X^{-bbar} * mu * sum_j X^j)
    {
        const uint32_t e = (2048u - abar[n]) & 2047u;
        for (int j = t; j < 1024; j += 64) {
            acc[0][j] = 0;
            const uint32_t idx = (uint32_t)(j - (int)e) & 2047u;
            acc[1][j] = idx < 1024u ? mu : 0u - mu;
        }
    }
    const FwdTw tw = load_fwd_tw(tb.fwd, t);
    const double2 twt = tb.tw[t];  // psi^t (untwist factors formed on the fly)
    auto bar = [] {
        lpb_jitter();
        __syncthreads();
    };
    auto wbar = [] {
        lpb_jitter();
        __syncwarp();
    };
    int xs = 0;  // alternating cross-warp tile

    constexpr uint32_t HALF = 1u << (BGBIT - 1);
    constexpr uint32_t MASK = (1u << BGBIT) - 1;
    uint32_t OFF = 0;
#pragma unroll
    for (int q = 1; q <= L; q++)
        OFF += HALF << (32 - q * BGBIT);
    OFF += 1u << (31 - L * BGBIT);

    constexpr int ROWS = 2 * L;
    for (uint32_t i = 0; i < n; i++) {
        lpb_jitter();
        __syncthreads();
        const uint32_t a = abar[i];
        LPB_ASSERT(a < 2048u);
        if (a == 0)
            continue;
        double2 oA[8], oB[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            oA[q] = make_double2(0.0, 0.0);
            oB[q] = make_double2(0.0, 0.0);
        }
        const double2* bki = bkf + (size_t)i * ROWS * 2 * FFT_M;
#pragma unroll
        for (int c = 0; c < 2; c++) {
            uint32_t tmp[16];
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const int j = t + 64 * q;
                tmp[q] = rot_read(acc[c], a, j) - acc[c][j] + OFF;
                tmp[8 + q] = rot_read(acc[c], a, j + 512) - acc[c][j + 512] + OFF;
            }
#pragma unroll 1
            for (int p = 0; p < L; p++) {
                const double2* row = bki + (size_t)(c * L + p) * 2 * FFT_M;
                double2 BA[8], BB[8];
                const int sh = 32 - (p + 1) * BGBIT;
                double2 x[8];
#pragma unroll
                for (int q = 0; q < 8; q++)
                    x[q] = make_double2(digit_to_double((tmp[q] >> sh) & MASK, HALF),
                                        digit_to_double((tmp[8 + q] >> sh) & MASK, HALF));
                fft_forward(x, tw, xbuf[xs], xbuf[2], t, bar, wbar);
                xs ^= 1;
                // BK_i rows for this digit, loaded at MAC time (L2-resident): measured faster
                // than a register prefetch one transform ahead, which spills
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    BA[q] = ld_stream(row + q * 64 + t);
                    BB[q] = ld_stream(row + FFT_M + q * 64 + t);
                }
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    mac(oA[q], x[q], BA[q]);
                    mac(oB[q], x[q], BB[q]);
                }
            }
        }
        // both inverse transforms in lockstep: shared barriers, twice the ILP.  Tiles:
        // intra and cross exchanges alias xbuf[2] / xbuf[xs] (a CTA barrier separates them)
        {
            const InvTw itw = load_inv_tw(tb.inv, t);
            fft_inverse2(oA, oB, itw, xbuf[2], xbuf[xs], xbuf[2], xbuf[xs], t, bar, wbar);
        }
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int j = t + 64 * q;
            const double2 ut = untwist(twt, q);
            const double2 wa = cmul(oA[q], ut);
            const double2 wb = cmul(oB[q], ut);
            if constexpr (ERR)
                emax = fmax(emax, fmax(fmax(fabs(wa.x - rint(wa.x)), fabs(wa.y - rint(wa.y))),
                                       fmax(fabs(wb.x - rint(wb.x)), fabs(wb.y - rint(wb.y)))));
            constexpr bool SAFE = kMagicRound<L, BGBIT>;
            acc[0][j] += round_low32<SAFE>(wa.x);
            acc[0][j + 512] += round_low32<SAFE>(wa.y);
            acc[1][j] += round_low32<SAFE>(wb.x);
            acc[1][j + 512] += round_low32<SAFE>(wb.y);
        }
    }
    __syncthreads();
    // ---- sample extraction at index 0 (N-dim LWE under the TRLWE key)
    uint32_t* o = pool_N + (size_t)it.out * dp.N_stride;
    for (int j = t; j < 1024; j += 64)
        o[j] = j == 0 ? acc[0][0] : 0u - acc[0][1024 - j];
    if (t == 0)
        o[1024] = acc[1][0];
    if constexpr (ERR)  // positive doubles order like their bit patterns
        atomicMax(err_out, (unsigned long long)__double_as_longlong(emax));
}

// ---------------------------------------------------------------------------
// K2: key switching.  KS_CT ciphertexts per CTA share every KSK row load; each
// thread owns KS_COLS consecutive output columns (one 16-byte load per row).
// The 2-bit digits (t = 8, basebit = 2) of the combined N-dim mask are staged in
// shared memory, one u16 per coefficient; a digit is the same for every lane of a
// warp (all lanes work on the same ciphertext), so the row choice is a
// warp-uniform branch and each selected row costs one add per column.
// ---------------------------------------------------------------------------
#ifndef KS_JUNROLL
#define KS_JUNROLL 1
#endif
constexpr int kKsJUnroll = KS_JUNROLL;  // digit-position loop unrolling (icache vs ILP)
#ifndef KS_PREFETCH
#define KS_PREFETCH 1
#endif
#ifndef KS_MINB
#define KS_MINB 4
#endif
#ifndef KS_CT_DEF
#define KS_CT_DEF 16
#endif
constexpr int KS_CT = KS_CT_DEF;
constexpr int KS_COLS = 4;
constexpr int KS_THREADS = 160;  // 640 columns >= n_stride

__global__ void __launch_bounds__(KS_THREADS, KS_MINB)
    k_keyswitch(DevParams dp, const KsItem* __restrict__ items, uint32_t count,
                const uint32_t* __restrict__ pool_N, uint32_t* __restrict__ pool_n,
                const uint32_t* __restrict__ ksk)
{
    extern __shared__ uint16_t dig[];  // [N][KS_CT]
    __shared__ uint32_t body[KS_CT];
    const uint32_t N = dp.N;
    const uint32_t first = blockIdx.x * KS_CT;
    const uint32_t nct = min((uint32_t)KS_CT, count - first);
    const uint32_t prec = 1u << (32 - (1 + dp.basebit * dp.t));

    for (uint32_t e = threadIdx.x; e < KS_CT * N; e += blockDim.x) {
        const uint32_t c = e / N, i = e - c * N;
        uint16_t d = 0;
        if (c < nct) {
            const KsItem it = items[first + c];
            LPB_ASSERT(it.in0 < dp.scratch_slots && it.out < dp.pool_slots &&
                       (it.in1 == SLOT_NONE || it.in1 < dp.scratch_slots));
            uint32_t v = pool_N[(size_t)it.in0 * dp.N_stride + i];
            if (it.in1 != SLOT_NONE)
                v += pool_N[(size_t)it.in1 * dp.N_stride + i];
            d = (uint16_t)((v + prec) >> 16);
        }
        dig[i * KS_CT + c] = d;
    }
    if (threadIdx.x < KS_CT) {
        uint32_t b = 0;
        if (threadIdx.x < nct) {
            const KsItem it = items[first + threadIdx.x];
            b = pool_N[(size_t)it.in0 * dp.N_stride + N] + it.off;
            if (it.in1 != SLOT_NONE)
                b += pool_N[(size_t)it.in1 * dp.N_stride + N];
        }
        body[threadIdx.x] = b;
    }
    __syncthreads();

    const uint32_t col = threadIdx.x * KS_COLS;
    if (col >= dp.n_stride)
        return;
    uint4 acc[KS_CT];
#pragma unroll
    for (int c = 0; c < KS_CT; c++) {
        acc[c] = make_uint4(0u, 0u, 0u, 0u);
        if (col + 0 == dp.n) acc[c].x = body[c];
        if (col + 1 == dp.n) acc[c].y = body[c];
        if (col + 2 == dp.n) acc[c].z = body[c];
        if (col + 3 == dp.n) acc[c].w = body[c];
    }
    const size_t row_stride = dp.n_stride;
    const uint4* base = reinterpret_cast<const uint4*>(ksk + col);
    const size_t rs4 = row_stride / 4;
#if KS_PREFETCH
    uint4 n1 = __ldg(base), n2 = __ldg(base + rs4), n3 = __ldg(base + 2 * rs4);
#endif
    for (uint32_t i = 0; i < N; i++) {
        uint32_t dw[KS_CT / 2];
        const uint32_t* dp32 = reinterpret_cast<const uint32_t*>(dig + i * KS_CT);
#pragma unroll
        for (int c = 0; c < KS_CT / 2; c++)
            dw[c] = dp32[c];  // broadcast: two ciphertexts' digit words
#pragma unroll kKsJUnroll
        for (int j = 0; j < 8; j++) {
#if KS_PREFETCH
            // rows of step (i, j) were loaded one step ahead; issue step (i, j+1) now
            const uint4 r1 = n1, r2 = n2, r3 = n3;
            {
                const uint32_t ni = j == 7 ? min(i + 1, N - 1) : i;
                const uint4* rn = base + ((size_t)ni * 24 + ((j + 1) & 7) * 3) * rs4;
                n1 = __ldg(rn);
                n2 = __ldg(rn + rs4);
                n3 = __ldg(rn + 2 * rs4);
            }
#else
            const uint4* rj = base + ((size_t)i * 24 + j * 3) * rs4;
            const uint4 r1 = __ldg(rj), r2 = __ldg(rj + rs4), r3 = __ldg(rj + 2 * rs4);
#endif
#pragma unroll
            for (int c = 0; c < KS_CT; c++) {
                const uint32_t w = dw[c >> 1] >> ((c & 1) * 16);
                const uint32_t d = (w >> (14 - 2 * j)) & 3u;
                if (d == 1) {
                    acc[c].x -= r1.x; acc[c].y -= r1.y; acc[c].z -= r1.z; acc[c].w -= r1.w;
                } else if (d == 2) {
                    acc[c].x -= r2.x; acc[c].y -= r2.y; acc[c].z -= r2.z; acc[c].w -= r2.w;
                } else if (d == 3) {
                    acc[c].x -= r3.x; acc[c].y -= r3.y; acc[c].z -= r3.z; acc[c].w -= r3.w;
                }
            }
        }
    }
#pragma unroll
    for (int c = 0; c < KS_CT; c++) {
        if ((uint32_t)c < nct) {
            const KsItem it = items[first + c];
            *reinterpret_cast<uint4*>(pool_n + (size_t)it.out * dp.n_stride + col) = acc[c];
        }
    }
}

// ---------------------------------------------------------------------------
// K3: free gates.
// ---------------------------------------------------------------------------
__global__ void k_linear(DevParams dp, const LinItem* __restrict__ items, uint32_t count,
                         uint32_t* __restrict__ pool_n)
{
    const uint32_t words = dp.n + 1;
    const uint64_t total = (uint64_t)count * words;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t g = (uint32_t)(e / words), w = (uint32_t)(e - (uint64_t)g * words);
        const LinItem it = items[g];
        LPB_ASSERT(it.out < dp.pool_slots && (it.kind == 2 || it.in0 < dp.pool_slots));
        uint32_t v;
        if (it.kind == 2)
            v = w == dp.n ? it.in0 : 0u;
        else {
            v = pool_n[(size_t)it.in0 * dp.n_stride + w];
            if (it.kind == 0)
                v = 0u - v;
        }
        pool_n[(size_t)it.out * dp.n_stride + w] = v;
    }
}

// Host-to-pool repack: packed wire rows (n+1 words) staged by one 1-D copy -> pitched pool
// rows.  A pinned 2-D copy with a 2,524 B row / 2,528 B pitch runs at ~19 GB/s on the
// B200 host link against ~55 GB/s for the 1-D copy (tools/copy_bench.py).
__global__ void k_repack_rows(DevParams dp, const uint32_t* __restrict__ packed, uint64_t count,
                              uint32_t* __restrict__ pool_rows)
{
    const uint32_t words = dp.n + 1;
    const uint64_t total = count * words;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = e / words, w = e - g * words;
        pool_rows[g * dp.n_stride + w] = packed[e];
    }
}

// Pool-to-host pack: pitched pool rows -> packed wire rows for one 1-D device-to-host copy.
__global__ void k_pack_rows(DevParams dp, const uint32_t* __restrict__ pool_rows, uint64_t count,
                            uint32_t* __restrict__ packed)
{
    const uint32_t words = dp.n + 1;
    const uint64_t total = count * words;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = e / words, w = e - g * words;
        packed[e] = pool_rows[g * dp.n_stride + w];
    }
}

// Wire payloads.  QUERY: [u8 l][l samples][u8 l][l samples]; samples are
// n+1 little-endian u32 (mask then body, torus.hpp:226-237), unaligned after the prefix.
__global__ void k_unpack_queries(DevParams dp, const uint8_t* __restrict__ bytes,
                                 const uint64_t* __restrict__ offs,
                                 const uint32_t* __restrict__ xf, const uint32_t* __restrict__ yf,
                                 uint64_t count, uint32_t l, uint32_t* __restrict__ pool_n)
{
    const uint32_t words = dp.n + 1;
    const uint64_t S = 4ull * words, per_q = 2ull * l * words;
    const uint64_t total = count * per_q;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t q = e / per_q, r = e - q * per_q;
        const uint32_t wsel = (uint32_t)(r / ((uint64_t)l * words));
        const uint64_t r2 = r - (uint64_t)wsel * l * words;
        const uint32_t i = (uint32_t)(r2 / words), k = (uint32_t)(r2 - (uint64_t)i * words);
        const uint8_t* src = bytes + offs[q] + wsel * (1 + l * S) + 1 + i * S + 4ull * k;
        const uint32_t v = (uint32_t)src[0] | ((uint32_t)src[1] << 8) | ((uint32_t)src[2] << 16) |
                           ((uint32_t)src[3] << 24);
        const uint32_t slot = (wsel ? yf[q] : xf[q]) + i;
        pool_n[(size_t)slot * dp.n_stride + k] = v;
    }
}

// ZEROSHEET rows (aligned, packed) + preprocess_services: body += encode_bit(bit).
__global__ void k_load_zero_sheet(DevParams dp, const uint32_t* __restrict__ sheet,
                                  const uint64_t* __restrict__ values, uint32_t bits,
                                  uint64_t regions, uint32_t first, uint32_t* __restrict__ pool_n)
{
    const uint32_t words = dp.n + 1;
    const uint64_t total = regions * bits * words;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = e / words, k = e - g * words;
        uint32_t v = sheet[e];
        if (k == dp.n) {
            const uint64_t r = g / bits, j = g - r * bits;
            v += ((values[r] >> j) & 1) ? 0x20000000u : 0xE0000000u;
        }
        pool_n[(first + g) * dp.n_stride + k] = v;
    }
}

// RESPONSE rows of several queries -> packed samples for one device-to-host copy.
__global__ void k_pack_responses(DevParams dp, const uint32_t* __restrict__ pool_n,
                                 const uint32_t* __restrict__ out_first, uint64_t count,
                                 uint32_t m, uint32_t* __restrict__ packed)
{
    const uint32_t words = dp.n + 1;
    const uint64_t total = count * m * words;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = e / words, k = e - g * words;
        const uint64_t q = g / m, j = g - q * m;
        packed[e] = pool_n[((size_t)out_first[q] + j) * dp.n_stride + k];
    }
}

// Counter-based client encryption (cbrng.h): one warp per sample; lanes
// generate Philox blocks of 4 mask words, the <a, key> sum is reduced mod 2^32 across
// the warp (order-free), lane 0 adds mu and the Box-Muller noise.
__global__ void k_client_encrypt(DevParams dp, const uint8_t* __restrict__ key, uint64_t seed,
                                 uint32_t first_index, const uint32_t* __restrict__ mus,
                                 uint64_t count, double alpha, uint64_t first_slot,
                                 uint32_t* __restrict__ pool_n)
{
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint32_t n = dp.n, blocks = (n + 3) / 4;
    for (uint64_t j = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < count;
         j += warps) {
        const uint32_t idx = first_index + (uint32_t)j;
        uint32_t* o = pool_n + (first_slot + j) * dp.n_stride;
        uint32_t dot = 0;
        for (uint32_t b = lane; b < blocks; b += 32) {
            const uint32_t ctr[4] = {idx, b, 0u, 0u};
            uint32_t r[4];
            cb_philox(ctr, seed, r);
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const uint32_t i = 4 * b + q;
                if (i < n) {
                    o[i] = r[q];
                    dot += r[q] * (uint32_t)key[i];
                }
            }
        }
#pragma unroll
        for (int off = 16; off; off >>= 1)
            dot += __shfl_xor_sync(0xFFFFFFFFu, dot, off);
        if (lane == 0)
            o[n] = dot + mus[j] + cb_noise(seed, idx, alpha);
    }
}

// FP64 FMA throughput probe (roofline denominator).
__global__ void k_fp64_peak(double* out, int iters)
{
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
    double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < iters; i++) {
        a0 = __fma_rn(a0, b, c); a1 = __fma_rn(a1, b, c); a2 = __fma_rn(a2, b, c);
        a3 = __fma_rn(a3, b, c); a4 = __fma_rn(a4, b, c); a5 = __fma_rn(a5, b, c);
        a6 = __fma_rn(a6, b, c); a7 = __fma_rn(a7, b, c);
    }
    const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678)
        out[0] = s;
}

}  // namespace lpb

namespace lpb {

// ---------------------------------------------------------------------------
// Small-batch (latency) kernels, used when a circuit level has fewer bootstraps
// than SMs (e.g. a single LocPIR query, BASELINE configs[0]).
// ---------------------------------------------------------------------------

// K2s: key switching split over KS_SPLIT coefficient ranges per ciphertext; the
// partial sums (mod 2^32, order-free, so bit-exact) are reduced by k_ks_reduce.
constexpr int KS_SPLIT = 32;

__global__ void __launch_bounds__(KS_THREADS)
    k_keyswitch_split(DevParams dp, const KsItem* __restrict__ items,
                      const uint32_t* __restrict__ pool_N, const uint32_t* __restrict__ ksk,
                      uint32_t* __restrict__ partial)
{
    const uint32_t g = blockIdx.x, split = blockIdx.y;
    const KsItem it = items[g];
    LPB_ASSERT(it.in0 < dp.scratch_slots && (it.in1 == SLOT_NONE || it.in1 < dp.scratch_slots));
    const uint32_t N = dp.N, per = N / KS_SPLIT;
    const uint32_t prec = 1u << (32 - (1 + dp.basebit * dp.t));
    const uint32_t col = threadIdx.x * KS_COLS;
    if (col >= dp.n_stride)
        return;
    const uint32_t* a0 = pool_N + (size_t)it.in0 * dp.N_stride;
    const uint32_t* a1 = it.in1 != SLOT_NONE ? pool_N + (size_t)it.in1 * dp.N_stride : nullptr;
    const size_t rs4 = dp.n_stride / 4;
    const uint4* base = reinterpret_cast<const uint4*>(ksk + col);
    uint4 acc = make_uint4(0u, 0u, 0u, 0u);
    for (uint32_t i = split * per; i < (split + 1) * per; i++) {
        uint32_t v = __ldg(a0 + i);
        if (a1)
            v += __ldg(a1 + i);
        const uint32_t w = (v + prec) >> 16;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint32_t d = (w >> (14 - 2 * j)) & 3u;
            if (d) {
                const uint4 r = __ldg(base + ((size_t)i * 24 + j * 3 + (d - 1)) * rs4);
                acc.x -= r.x;
                acc.y -= r.y;
                acc.z -= r.z;
                acc.w -= r.w;
            }
        }
    }
    *reinterpret_cast<uint4*>(partial + ((size_t)g * KS_SPLIT + split) * dp.n_stride + col) = acc;
}

__global__ void __launch_bounds__(KS_THREADS)
    k_ks_reduce(DevParams dp, const KsItem* __restrict__ items,
                const uint32_t* __restrict__ pool_N, const uint32_t* __restrict__ partial,
                uint32_t* __restrict__ pool_n)
{
    const uint32_t g = blockIdx.x;
    const KsItem it = items[g];
    LPB_ASSERT(it.out < dp.pool_slots);
    for (uint32_t col = threadIdx.x; col < dp.n_stride; col += blockDim.x) {
        uint32_t v = 0;
        if (col == dp.n) {
            v = pool_N[(size_t)it.in0 * dp.N_stride + dp.N] + it.off;
            if (it.in1 != SLOT_NONE)
                v += pool_N[(size_t)it.in1 * dp.N_stride + dp.N];
        }
        for (int s = 0; s < KS_SPLIT; s++)
            v += partial[((size_t)g * KS_SPLIT + s) * dp.n_stride + col];
        pool_n[(size_t)it.out * dp.n_stride + col] = v;
    }
}

// K1l: blind rotation with the 2l digit transforms of one ciphertext in parallel,
// one 64-thread group each (named barrier per group); the frequency-domain MAC runs
// in the oracle's row order (rows 0..2l-1, same fma chain), so results stay
// bit-exact; groups 0 and 1 then run the two inverse transforms in parallel.
template <int L>
struct LatSmem {
    uint32_t acc[2][1024];
    double2 F[2 * L][FFT_M];              // digit spectra, slot layout [q*64 + t]
    double2 O[2][FFT_M];                  // MAC results per output component
    double2 tiles[2 * L][2][XTILE];       // per group: cross-warp tile, intra-warp tile
    uint16_t abar[MAX_N + 1];
};
template <int L>
constexpr size_t kLatSmemBytes = sizeof(LatSmem<L>);

__device__ __forceinline__ void group_bar(int id)
{
    lpb_jitter();
    asm volatile("bar.sync %0, 64;\n" ::"r"(id) : "memory");
}

template <int L, int BGBIT>
__global__ void __launch_bounds__(128 * L, 1)
    k_blind_rotate_lat(DevParams dp, const BrItem* __restrict__ items,
                       const uint32_t* __restrict__ pool_n, uint32_t* __restrict__ pool_N,
                       const double2* __restrict__ bkf, FftTabs tb, uint32_t mu)
{
    extern __shared__ __align__(16) uint8_t smem_l[];
    LatSmem<L>& S = *reinterpret_cast<LatSmem<L>*>(smem_l);
    const int g = threadIdx.x >> 6, t = threadIdx.x & 63;
    const BrItem it = items[blockIdx.x];
    const uint32_t n = dp.n;
    LPB_ASSERT(it.out < dp.scratch_slots && n <= MAX_N);
    lpb_poison_smem(smem_l, sizeof(LatSmem<L>));
    {
        const uint32_t* a0 = lwe_row(dp, pool_n, it.in0);
        const uint32_t* a1 = it.in1 != SLOT_NONE ? lwe_row(dp, pool_n, it.in1) : nullptr;
        const uint32_t* a2 = it.in2 != SLOT_NONE ? lwe_row(dp, pool_n, it.in2) : nullptr;
        for (uint32_t i = threadIdx.x; i <= n; i += blockDim.x) {
            uint32_t v = (uint32_t)it.c0 * a0[i];
            if (a1)
                v += (uint32_t)it.c1 * a1[i];
            if (a2)
                v += (uint32_t)it.c2 * a2[i];
            if (i == n)
                v += it.off;
            S.abar[i] = (uint16_t)((v + (1u << 20)) >> 21);
        }
    }
    __syncthreads();
    {
        const uint32_t e = (2048u - S.abar[n]) & 2047u;
        for (int j = threadIdx.x; j < 1024; j += blockDim.x) {
            S.acc[0][j] = 0;
            const uint32_t idx = (uint32_t)(j - (int)e) & 2047u;
            S.acc[1][j] = idx < 1024u ? mu : 0u - mu;
        }
    }
    const FwdTw ftw = load_fwd_tw(tb.fwd, t);
    const double2 twt = tb.tw[t];
    const int bid = 1 + g;
    auto bar = [bid] { group_bar(bid); };
    auto wbar = [] { __syncwarp(); };
    constexpr uint32_t HALF = 1u << (BGBIT - 1);
    constexpr uint32_t MASK = (1u << BGBIT) - 1;
    uint32_t OFF = 0;
#pragma unroll
    for (int q = 1; q <= L; q++)
        OFF += HALF << (32 - q * BGBIT);
    OFF += 1u << (31 - L * BGBIT);
    constexpr int ROWS = 2 * L;
    const int c = g / L, p = g % L;
    const int sh = 32 - (p + 1) * BGBIT;

    // MAC split over all 2L groups: group g serves output component g / L and the
    // frequency slots q*64 + t with q = g % L + L*k (at most P of them per thread); each
    // slot's chain over the 2L rows keeps the oracle's order, so the result is unchanged.
    // L = 2: each thread serves BOTH output components for slots q = g, g + 4, so every
    // digit-spectrum element is read from shared memory once.  L = 3 (384 threads, at the
    // register limit): each thread serves output component g / L for q = g % L + L k.
    constexpr bool BOTH = (L == 2);
    constexpr int P = BOTH ? 2 : (8 + L - 1) / L;
    constexpr int NO = BOTH ? 2 : 1;  // output components per thread
    const int mcomp = g / L, msub = g % L;
    auto slot_q = [&](int k) { return BOTH ? g + 2 * L * k : msub + L * k; };
#ifdef LPB_PHASE_CLK
    // diagnostic build only: per-phase clock sums of thread 0 of CTA 0
    unsigned long long ph[12] = {0}, tp = clock64();
    auto mark = [&](int k) {
        const unsigned long long now = clock64();
        ph[k] += now - tp;
        tp = now;
    };
#else
    auto mark = [](int) {};
#endif
    for (uint32_t i = 0; i < n; i++) {
        __syncthreads();
        mark(0);
        const uint32_t a = S.abar[i];
        if (a == 0)
            continue;
        // this thread's BK values for its MAC slots, in flight during the transform
        double2 bkv[ROWS][NO][P];
        const double2* bki = bkf + (size_t)i * ROWS * 2 * FFT_M;
        auto load_rows = [&](int r0, int r1) {
#pragma unroll
            for (int r = r0; r < r1; r++)
#pragma unroll
                for (int o = 0; o < NO; o++)
#pragma unroll
                    for (int k = 0; k < P; k++) {
                        const int q = slot_q(k);
                        const int comp = BOTH ? o : mcomp;
                        if (q < 8)
                            bkv[r][o][k] = ld_stream(bki + ((size_t)r * 2 + comp) * FFT_M + q * 64 + t);
                    }
        };
        // l = 3: the BK loads are issued in thirds AFTER the digit reads and each exchange,
        // so they drain through L1TEX during the FP64 passes instead of queueing in front
        // of the rotated ACC reads (K1l launch 2.30 -> 2.23 ms); l = 2: all up front
        // (spreading them measured 1.27 -> 1.36 ms).  tools/r3_k1l_ab.sh
        constexpr bool SPREAD = LAT_BK_SPREAD && L == 3;
        constexpr int B0 = SPREAD ? LAT_BK_B0 : ROWS;
        constexpr int B1 = SPREAD ? (LAT_BK_B1 < ROWS ? LAT_BK_B1 : ROWS) : ROWS;
        if constexpr (!SPREAD)
            load_rows(0, ROWS);
        // every group: digit (c, p) of (X^a - 1) ACC_c -> forward transform -> F[g]
        {
            double2 x[8];
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const int j = t + 64 * q;
                const uint32_t lo = rot_read(S.acc[c], a, j) - S.acc[c][j] + OFF;
                const uint32_t hi = rot_read(S.acc[c], a, j + 512) - S.acc[c][j + 512] + OFF;
                x[q] = make_double2(digit_to_double((lo >> sh) & MASK, HALF),
                                    digit_to_double((hi >> sh) & MASK, HALF));
            }
            mark(6);
            if constexpr (SPREAD)
                load_rows(0, B0);
            fwd_pass0(x);
            mark(7);
            exch_p0_to_p1(x, S.tiles[g][0], t, bar);
            mark(8);
            if constexpr (SPREAD)
                load_rows(B0, B1);
            fwd_pass1(x, ftw);
            mark(9);
            exch_p1_to_p2(x, S.tiles[g][1], t, wbar);
            mark(10);
            if constexpr (SPREAD)
                load_rows(B1, ROWS);
            fwd_pass2(x, ftw);
            mark(11);
#pragma unroll
            for (int q = 0; q < 8; q++)
                S.F[g][q * 64 + t] = x[q];
        }
        mark(1);
        __syncthreads();
        mark(2);
#pragma unroll
        for (int k = 0; k < P; k++) {
            const int q = slot_q(k);
            if (q < 8) {
                double2 oo[NO];
#pragma unroll
                for (int o = 0; o < NO; o++)
                    oo[o] = make_double2(0.0, 0.0);
#pragma unroll
                for (int r = 0; r < ROWS; r++) {
                    const double2 F = S.F[r][q * 64 + t];
#pragma unroll
                    for (int o = 0; o < NO; o++)
                        mac(oo[o], F, bkv[r][o][k]);
                }
#pragma unroll
                for (int o = 0; o < NO; o++)
                    S.O[BOTH ? o : mcomp][q * 64 + t] = oo[o];
            }
        }
        mark(3);
        __syncthreads();
        mark(4);
        // groups 0 / 1: inverse transform of output component g, ACC update
        if (g < 2) {
            const int comp = g;
            double2 o[8];
#pragma unroll
            for (int q = 0; q < 8; q++)
                o[q] = S.O[comp][q * 64 + t];
            const InvTw itw = load_inv_tw(tb.inv, t);
            fft_inverse(o, itw, S.tiles[g][0], S.tiles[g][1], t, bar, wbar);
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const int j = t + 64 * q;
                const double2 w = cmul(o[q], untwist(twt, q));
                S.acc[comp][j] += round_low32<kMagicRound<L, BGBIT>>(w.x);
                S.acc[comp][j + 512] += round_low32<kMagicRound<L, BGBIT>>(w.y);
            }
        }
        mark(5);
    }
#ifdef LPB_PHASE_CLK
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("K1l<%d> phase clocks per step (n=%u): top-barrier %.0f fwd %.0f fwd-barrier %.0f "
               "mac %.0f mac-barrier %.0f inverse %.0f\n", L, n, ph[0] / (double)n, ph[1] / (double)n,
               ph[2] / (double)n, ph[3] / (double)n, ph[4] / (double)n, ph[5] / (double)n);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        printf("  fwd split: digits %.0f pass0 %.0f xchg1 %.0f pass1 %.0f xchg2 %.0f pass2 %.0f\n",
               ph[6] / (double)n, ph[7] / (double)n, ph[8] / (double)n, ph[9] / (double)n,
               ph[10] / (double)n, ph[11] / (double)n);
#endif
    __syncthreads();
    uint32_t* out = pool_N + (size_t)it.out * dp.N_stride;
    for (int j = threadIdx.x; j < 1024; j += blockDim.x)
        out[j] = j == 0 ? S.acc[0][0] : 0u - S.acc[0][1024 - j];
    if (threadIdx.x == 0)
        out[1024] = S.acc[1][0];
}

}  // namespace lpb
