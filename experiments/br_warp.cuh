// br_warp.cuh -- warp-per-ciphertext blind rotation (K1w) for sm_100a.
//
// Same algorithm and the same FP64 operations as k_blind_rotate / the oracle
// (radix-2 DIF forward, radix-2 DIT inverse, oracle twiddle tables, oracle fma
// patterns), regrouped so that one warp owns one ciphertext:
//   * 16 complex points per lane; the 512-point transform is 4 radix-2 stages in
//     registers (pass A: positions t + 32q), ONE shared-memory exchange inside the
//     warp, 4 more in-register stages (pass B: lane L = 2b + e holds positions
//     32b + 2q + e), and the last stage across lane pairs with one shuffle swap
//     (its twiddle is exactly 1).  No CTA barrier anywhere in the main loop.
//   * The frequency-domain accumulators, the twist factors and the per-lane
//     twiddles live in TMEM (tcgen05.ld/st, a data path separate from shared
//     memory), freeing registers for 16-point lanes.
//   * The BK is stored slot-major in lane order ([q][L]) so each load instruction
//     reads 512 contiguous bytes.
// CTA = 4 warps (one per TMEM lane quarter) = 4 ciphertexts; 256 TMEM columns per CTA.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft.cuh"

namespace lpb {

constexpr int W_CT = 4;            // ciphertexts (warps) per CTA
constexpr int WTILE = 16 * 34;     // exchange tile: position 32a + c at slot 34a + c
// TMEM columns per lane
constexpr size_t W_SMEM = (size_t)W_CT * (WTILE * 16 + 2048 * 4 + (MAX_N + 1) * 2);
constexpr uint32_t TM_OUTA = 0, TM_OUTB = 64, TM_TWIST = 128, TM_TWA = 192, TM_TWB = 224;

__device__ __forceinline__ void tm_ld32(uint32_t addr, uint32_t (&v)[32])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void tm_st32(uint32_t addr, const uint32_t (&v)[32])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
        "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n"
        :
        : "r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]),
          "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]),
          "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]),
          "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
          "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}

__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ double2 u2d(const uint32_t* v)
{
    return make_double2(__hiloint2double((int)v[1], (int)v[0]), __hiloint2double((int)v[3], (int)v[2]));
}
__device__ __forceinline__ void d2u(uint32_t* v, double2 d)
{
    v[0] = (uint32_t)__double2loint(d.x);
    v[1] = (uint32_t)__double2hiint(d.x);
    v[2] = (uint32_t)__double2loint(d.y);
    v[3] = (uint32_t)__double2hiint(d.y);
}

// 8 complex values <-> TMEM columns [col, col + 32)
__device__ __forceinline__ void tm_load8(uint32_t addr, double2 (&d)[8])
{
    uint32_t v[32];
    tm_ld32(addr, v);
#pragma unroll
    for (int q = 0; q < 8; q++)
        d[q] = u2d(v + 4 * q);
}
__device__ __forceinline__ void tm_store8(uint32_t addr, const double2* d)
{
    uint32_t v[32];
#pragma unroll
    for (int q = 0; q < 8; q++)
        d2u(v + 4 * q, d[q]);
    tm_st32(addr, v);
}

// ---- pass A: lane t holds positions t + 32 q, q = 0..15 (DIF stages 0..3) ---------
// twA: W[t], W[t+32], W[t+64], W[t+96], W[2t], W[2t+64], W[4t], W[8t]
__device__ __forceinline__ void passA_fwd(double2 (&x)[16], const double2 (&w)[8])
{
#pragma unroll
    for (int q = 0; q < 8; q++)
        dif(x[q], x[q + 8], q < 4 ? w[q] : mul_i(w[q - 4]));
#pragma unroll
    for (int g = 0; g < 16; g += 8)
#pragma unroll
        for (int m = 0; m < 4; m++)
            dif(x[g + m], x[g + m + 4], m < 2 ? w[4 + m] : mul_i(w[4 + m - 2]));
#pragma unroll
    for (int g = 0; g < 16; g += 4) {
        dif(x[g], x[g + 2], w[6]);
        dif(x[g + 1], x[g + 3], mul_i(w[6]));
    }
#pragma unroll
    for (int q = 0; q < 16; q += 2)
        dif(x[q], x[q + 1], w[7]);
}

__device__ __forceinline__ void passA_inv(double2 (&x)[16], const double2 (&w)[8])
{
#pragma unroll
    for (int q = 0; q < 16; q += 2)
        dit(x[q], x[q + 1], conj2(w[7]));
#pragma unroll
    for (int g = 0; g < 16; g += 4) {
        dit(x[g], x[g + 2], conj2(w[6]));
        dit(x[g + 1], x[g + 3], conj2(mul_i(w[6])));
    }
#pragma unroll
    for (int g = 0; g < 16; g += 8)
#pragma unroll
        for (int m = 0; m < 4; m++)
            dit(x[g + m], x[g + m + 4], conj2(m < 2 ? w[4 + m] : mul_i(w[4 + m - 2])));
#pragma unroll
    for (int q = 0; q < 8; q++)
        dit(x[q], x[q + 8], conj2(q < 4 ? w[q] : mul_i(w[q - 4])));
}

// ---- pass B: lane L = 2b + e holds positions 32b + 2q + e (DIF stages 4..7) --------
// twB: W[16e], W[16e+32], W[16e+64], W[16e+96], W[32e], W[64+32e], W[64e], W[128e]
__device__ __forceinline__ void passB_fwd(double2 (&x)[16], const double2 (&w)[8])
{
#pragma unroll
    for (int q = 0; q < 8; q++)
        dif(x[q], x[q + 8], q < 4 ? w[q] : mul_i(w[q - 4]));
#pragma unroll
    for (int g = 0; g < 16; g += 8)
#pragma unroll
        for (int m = 0; m < 4; m++)
            dif(x[g + m], x[g + m + 4], m < 2 ? w[4 + m] : mul_i(w[4 + m - 2]));
#pragma unroll
    for (int g = 0; g < 16; g += 4) {
        dif(x[g], x[g + 2], w[6]);
        dif(x[g + 1], x[g + 3], mul_i(w[6]));
    }
#pragma unroll
    for (int q = 0; q < 16; q += 2)
        dif(x[q], x[q + 1], w[7]);
}

__device__ __forceinline__ void passB_inv(double2 (&x)[16], const double2 (&w)[8])
{
#pragma unroll
    for (int q = 0; q < 16; q += 2)
        dit(x[q], x[q + 1], conj2(w[7]));
#pragma unroll
    for (int g = 0; g < 16; g += 4) {
        dit(x[g], x[g + 2], conj2(w[6]));
        dit(x[g + 1], x[g + 3], conj2(mul_i(w[6])));
    }
#pragma unroll
    for (int g = 0; g < 16; g += 8)
#pragma unroll
        for (int m = 0; m < 4; m++)
            dit(x[g + m], x[g + m + 4], conj2(m < 2 ? w[4 + m] : mul_i(w[4 + m - 2])));
#pragma unroll
    for (int q = 0; q < 8; q++)
        dit(x[q], x[q + 8], conj2(q < 4 ? w[q] : mul_i(w[q - 4])));
}

// ---- stage 8 (twiddle exactly 1) across lane pairs: lane e=0 keeps u + v, e=1 u - v.
__device__ __forceinline__ void stage8_pair(double2 (&x)[16], double sgn)
{
#pragma unroll
    for (int q = 0; q < 16; q++) {
        const double rx = __shfl_xor_sync(0xffffffffu, x[q].x, 1);
        const double ry = __shfl_xor_sync(0xffffffffu, x[q].y, 1);
        // e=0: own + recv = u + v;  e=1: recv - own = u - v   (single rounding each)
        x[q].x = __fma_rn(sgn, x[q].x, rx);
        x[q].y = __fma_rn(sgn, x[q].y, ry);
    }
}

// ---- exchanges inside the warp (slot 34a + c for position 32a + c) -----------------
__device__ __forceinline__ void exch_A_to_B(double2 (&x)[16], double2* tile, int lane)
{
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 16; q++)
        tile[34 * q + lane] = x[q];  // position lane + 32 q
    __syncwarp();
    const double2* rd = tile + 34 * (lane >> 1) + (lane & 1);
#pragma unroll
    for (int q = 0; q < 16; q++)
        x[q] = rd[2 * q];  // position 32 (lane>>1) + 2q + (lane&1)
}
__device__ __forceinline__ void exch_B_to_A(double2 (&x)[16], double2* tile, int lane)
{
    __syncwarp();
    double2* w = tile + 34 * (lane >> 1) + (lane & 1);
#pragma unroll
    for (int q = 0; q < 16; q++)
        w[2 * q] = x[q];
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 16; q++)
        x[q] = tile[34 * q + lane];
}

// K0w: BK torus polynomials -> frequency domain, slot-major lane order [q][L].
__global__ void __launch_bounds__(32 * W_CT) k_bk_to_freq_w(const uint32_t* __restrict__ bk,
                                                         double2* __restrict__ out,
                                                         const double2* __restrict__ W,
                                                         const double2* __restrict__ TW,
                                                         uint32_t polys)
{
    __shared__ __align__(16) double2 tiles[W_CT][WTILE];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t poly = (size_t)blockIdx.x * W_CT + warp;
    if (poly >= polys)
        return;
    const uint32_t* b = bk + poly * 1024;
    double2 wa[8], wb[8];
    const int e = lane & 1;
    wa[0] = W[lane]; wa[1] = W[lane + 32]; wa[2] = W[lane + 64]; wa[3] = W[lane + 96];
    wa[4] = W[2 * lane]; wa[5] = W[2 * lane + 64]; wa[6] = W[4 * lane]; wa[7] = W[8 * lane];
    wb[0] = W[16 * e]; wb[1] = W[16 * e + 32]; wb[2] = W[16 * e + 64]; wb[3] = W[16 * e + 96];
    wb[4] = W[32 * e]; wb[5] = W[64 + 32 * e]; wb[6] = W[64 * e]; wb[7] = W[128 * e];
    double2 x[16];
#pragma unroll
    for (int q = 0; q < 16; q++) {
        const int j = lane + 32 * q;
        x[q] = cmul(make_double2((double)(int32_t)b[j], (double)(int32_t)b[j + 512]), TW[j]);
    }
    passA_fwd(x, wa);
    exch_A_to_B(x, tiles[warp], lane);
    passB_fwd(x, wb);
    stage8_pair(x, e ? -1.0 : 1.0);
    double2* o = out + poly * FFT_M;
#pragma unroll
    for (int q = 0; q < 16; q++)
        o[q * 32 + lane] = x[q];
}

// K1w: blind rotation + sample extraction, one warp per ciphertext.
template <int L, int BGBIT>
__global__ void __launch_bounds__(32 * W_CT, 2)
    k_blind_rotate_w(DevParams dp, const BrItem* __restrict__ items, uint32_t count,
                     const uint32_t* __restrict__ pool_n, uint32_t* __restrict__ pool_N,
                     const double2* __restrict__ bkf, const double2* __restrict__ W,
                     const double2* __restrict__ TW, uint32_t mu)
{
    // dynamic smem: exchange tiles | ACC (2 x 1024 u32) | mod-switched mask, per warp
    extern __shared__ __align__(16) uint8_t smem_w[];
    double2* tiles = reinterpret_cast<double2*>(smem_w);
    uint32_t* accs = reinterpret_cast<uint32_t*>(smem_w + (size_t)W_CT * WTILE * 16);
    uint16_t* abars = reinterpret_cast<uint16_t*>(smem_w + (size_t)W_CT * WTILE * 16 +
                                                  (size_t)W_CT * 2048 * 4);
    __shared__ uint32_t tmem_slot;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int e = lane & 1;
    const double sgn = e ? -1.0 : 1.0;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tb = tmem_slot + ((uint32_t)(warp * 32) << 16);
    const uint32_t item_idx = blockIdx.x * W_CT + warp;
    uint32_t* acc0 = accs + (size_t)warp * 2048;
    uint32_t* acc1 = acc0 + 1024;
    double2* tile = tiles + (size_t)warp * WTILE;
    uint16_t* abar = abars + (size_t)warp * (MAX_N + 1);

    if (item_idx < count) {
        const BrItem it = items[item_idx];
        const uint32_t n = dp.n;
        // per-lane constants into TMEM: twist (16), pass-A and pass-B twiddles (8 + 8)
        {
            double2 v[8];
#pragma unroll
            for (int h = 0; h < 2; h++) {
#pragma unroll
                for (int q = 0; q < 8; q++)
                    v[q] = TW[lane + 32 * (8 * h + q)];
                tm_store8(tb + TM_TWIST + 32 * h, v);
            }
            v[0] = W[lane]; v[1] = W[lane + 32]; v[2] = W[lane + 64]; v[3] = W[lane + 96];
            v[4] = W[2 * lane]; v[5] = W[2 * lane + 64]; v[6] = W[4 * lane]; v[7] = W[8 * lane];
            tm_store8(tb + TM_TWA, v);
            v[0] = W[16 * e]; v[1] = W[16 * e + 32]; v[2] = W[16 * e + 64]; v[3] = W[16 * e + 96];
            v[4] = W[32 * e]; v[5] = W[64 + 32 * e]; v[6] = W[64 * e]; v[7] = W[128 * e];
            tm_store8(tb + TM_TWB, v);
        }
        // gate linear form + mod switch (gate_engine.hpp:196-269)
        {
            const uint32_t* a0 = pool_n + (size_t)it.in0 * dp.n_stride;
            const uint32_t* a1 = it.in1 != SLOT_NONE ? pool_n + (size_t)it.in1 * dp.n_stride : nullptr;
            const uint32_t* a2 = it.in2 != SLOT_NONE ? pool_n + (size_t)it.in2 * dp.n_stride : nullptr;
            for (uint32_t i = lane; i <= n; i += 32) {
                uint32_t v = (uint32_t)it.c0 * a0[i];
                if (a1)
                    v += (uint32_t)it.c1 * a1[i];
                if (a2)
                    v += (uint32_t)it.c2 * a2[i];
                if (i == n)
                    v += it.off;
                abar[i] = (uint16_t)((v + (1u << 20)) >> 21);
            }
        }
        __syncwarp();
        {
            const uint32_t ee = (2048u - abar[n]) & 2047u;
            for (int j = lane; j < 1024; j += 32) {
                acc0[j] = 0;
                const uint32_t idx = (uint32_t)(j - (int)ee) & 2047u;
                acc1[j] = idx < 1024u ? mu : 0u - mu;
            }
        }
        tm_wait_st();

        constexpr uint32_t HALF = 1u << (BGBIT - 1);
        constexpr uint32_t MASK = (1u << BGBIT) - 1;
        uint32_t OFF = 0;
#pragma unroll
        for (int q = 1; q <= L; q++)
            OFF += HALF << (32 - q * BGBIT);
        OFF += 1u << (31 - L * BGBIT);
        constexpr int ROWS = 2 * L;

        for (uint32_t i = 0; i < n; i++) {
            __syncwarp();
            const uint32_t a = abar[i];
            if (a == 0)
                continue;
            const double2* bki = bkf + (size_t)i * ROWS * 2 * FFT_M;
#pragma unroll 1
            for (int c = 0; c < 2; c++) {
                const uint32_t* accc = c ? acc1 : acc0;
                uint32_t tmp[32];
#pragma unroll
                for (int q = 0; q < 16; q++) {
                    const int j = lane + 32 * q;
                    tmp[q] = rot_read(accc, a, j) - accc[j] + OFF;
                    tmp[16 + q] = rot_read(accc, a, j + 512) - accc[j + 512] + OFF;
                }
#pragma unroll 1
                for (int p = 0; p < L; p++) {
                    const int rr = c * L + p;
                    const int sh = 32 - (p + 1) * BGBIT;
                    // BK row rr, chunk k = (comp, h): 8 slots; chunk 0 is in flight during the FFT
                    const double2* row = bki + (size_t)rr * 2 * FFT_M + lane;
                    double2 Bn[8];
#pragma unroll
                    for (int q = 0; q < 8; q++)
                        Bn[q] = ld_stream(row + q * 32);
                    double2 x[16];
                    {
                        double2 tw[8];
#pragma unroll
                        for (int h = 0; h < 2; h++) {
                            tm_load8(tb + TM_TWIST + 32 * h, tw);
#pragma unroll
                            for (int q = 0; q < 8; q++) {
                                const int qq = 8 * h + q;
                                const int dlo = (int)((tmp[qq] >> sh) & MASK) - (int)HALF;
                                const int dhi = (int)((tmp[16 + qq] >> sh) & MASK) - (int)HALF;
                                x[qq] = cmul(make_double2((double)dlo, (double)dhi), tw[q]);
                            }
                        }
                    }
                    // passes A and B share one copy of the 4-stage code (I-cache)
#pragma unroll 1
                    for (int ps = 0; ps < 2; ps++) {
                        double2 w[8];
                        tm_load8(tb + (ps ? TM_TWB : TM_TWA), w);
                        passA_fwd(x, w);
                        if (ps == 0)
                            exch_A_to_B(x, tile, lane);
                    }
                    stage8_pair(x, sgn);
                    // MAC: OUT_comp[q] += F[q] * BK[rr][comp][q][lane], accumulators in TMEM
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        const int comp = k >> 1, h = k & 1;
                        double2 B[8], o[8];
#pragma unroll
                        for (int q = 0; q < 8; q++)
                            B[q] = Bn[q];
                        if (k < 3) {
                            const int kc = (k + 1) >> 1, kh = (k + 1) & 1;
#pragma unroll
                            for (int q = 0; q < 8; q++)
                                Bn[q] = ld_stream(row + kc * FFT_M + (8 * kh + q) * 32);
                        }
                        const uint32_t col = (comp ? TM_OUTB : TM_OUTA) + 32 * h;
                        if (rr > 0) {
                            tm_wait_st();
                            tm_load8(tb + col, o);
                        } else {
#pragma unroll
                            for (int q = 0; q < 8; q++)
                                o[q] = make_double2(0.0, 0.0);
                        }
#pragma unroll
                        for (int q = 0; q < 8; q++)
                            mac(o[q], x[8 * h + q], B[q]);
                        tm_store8(tb + col, o);
                    }
                }
            }
            tm_wait_st();
            // inverse transforms, round, accumulate into ACC
#pragma unroll 1
            for (int comp = 0; comp < 2; comp++) {
                double2 x[16];
                {
                    double2 o[8];
                    tm_load8(tb + (comp ? TM_OUTB : TM_OUTA), o);
#pragma unroll
                    for (int q = 0; q < 8; q++)
                        x[q] = o[q];
                    tm_load8(tb + (comp ? TM_OUTB : TM_OUTA) + 32, o);
#pragma unroll
                    for (int q = 0; q < 8; q++)
                        x[8 + q] = o[q];
                }
                stage8_pair(x, sgn);
#pragma unroll 1
                for (int ps = 0; ps < 2; ps++) {
                    double2 w[8];
                    tm_load8(tb + (ps ? TM_TWA : TM_TWB), w);
                    passA_inv(x, w);
                    if (ps == 0)
                        exch_B_to_A(x, tile, lane);
                }
                uint32_t* accc = comp ? acc1 : acc0;
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    double2 tw[8];
                    tm_load8(tb + TM_TWIST + 32 * h, tw);
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        const int j = lane + 32 * (8 * h + q);
                        const double2 w = cmul(x[8 * h + q], untwist(tw[q]));
                        accc[j] += (uint32_t)__double2ll_rn(w.x);
                        accc[j + 512] += (uint32_t)__double2ll_rn(w.y);
                    }
                }
            }
        }
        __syncwarp();
        uint32_t* o = pool_N + (size_t)it.out * dp.N_stride;
        for (int j = lane; j < 1024; j += 32)
            o[j] = j == 0 ? acc0[0] : 0u - acc0[1024 - j];
        if (lane == 0)
            o[1024] = acc1[0];
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem_slot));
}

}  // namespace lpb
