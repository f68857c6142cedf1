// br_pair.cuh -- blind rotation with paired digit transforms (K1p) for sm_100a.
//
// Same CTA shape as k_blind_rotate (64 threads per ciphertext, 8 points per thread)
// and the same FP64 operations in the same order (bit-exact with the oracle), but
// each thread transforms TWO digit polynomials in lockstep: they share every
// exchange barrier (half the CTA barriers per CMux step) and the compiler
// interleaves their independent butterflies (twice the ILP per warp).  To afford
// the second polynomial's registers, the frequency-domain accumulators live in
// TMEM between digit pairs (tcgen05.ld/st, 64 columns per CTA).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft.cuh"
#include "kernels.cuh"

namespace lpb {

struct PairSmem {
    uint32_t acc[2][1024];
    double2 tws[FFT_M];
    double2 cross[2][XTILE];
    double2 intra[2][XTILE];
    uint16_t abar[MAX_N + 1];
    uint32_t tmem_slot;
};

__device__ __forceinline__ void tm_mac_load(uint32_t addr, double2 (&o)[8])
{
    uint32_t v[32];
    tmem_ld32(addr, v);
#pragma unroll
    for (int q = 0; q < 8; q++)
        o[q] = unpack2(v + 4 * q);
}
__device__ __forceinline__ void tm_mac_store(uint32_t addr, const double2 (&o)[8])
{
    uint32_t v[32];
#pragma unroll
    for (int q = 0; q < 8; q++)
        pack2(v + 4 * q, o[q]);
    tmem_st32(addr, v);
}

template <int L, int BGBIT>
__global__ void __launch_bounds__(64, 4)
    k_blind_rotate_pair(DevParams dp, const BrItem* __restrict__ items,
                        const uint32_t* __restrict__ pool_n, uint32_t* __restrict__ pool_N,
                        const double2* __restrict__ bkf, const double2* __restrict__ W,
                        const double2* __restrict__ TW, uint32_t mu)
{
    extern __shared__ __align__(16) uint8_t smem_p[];
    PairSmem& S = *reinterpret_cast<PairSmem*>(smem_p);
    const int t = threadIdx.x;
    const BrItem it = items[blockIdx.x];
    const uint32_t n = dp.n;
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&S.tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    for (int j = t; j < FFT_M; j += 64)
        S.tws[j] = TW[j];
    {
        const uint32_t* a0 = pool_n + (size_t)it.in0 * dp.n_stride;
        const uint32_t* a1 = it.in1 != SLOT_NONE ? pool_n + (size_t)it.in1 * dp.n_stride : nullptr;
        const uint32_t* a2 = it.in2 != SLOT_NONE ? pool_n + (size_t)it.in2 * dp.n_stride : nullptr;
        for (uint32_t i = t; i <= n; i += 64) {
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
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tb = S.tmem_slot + ((uint32_t)(t & 32) << 16);
    {
        const uint32_t e = (2048u - S.abar[n]) & 2047u;
        for (int j = t; j < 1024; j += 64) {
            S.acc[0][j] = 0;
            const uint32_t idx = (uint32_t)(j - (int)e) & 2047u;
            S.acc[1][j] = idx < 1024u ? mu : 0u - mu;
        }
    }
    const Twiddles tw = load_twiddles(W, t);
    auto bar = [] { __syncthreads(); };
    auto wbar = [] { __syncwarp(); };

    constexpr uint32_t HALF = 1u << (BGBIT - 1);
    constexpr uint32_t MASK = (1u << BGBIT) - 1;
    uint32_t OFF = 0;
#pragma unroll
    for (int q = 1; q <= L; q++)
        OFF += HALF << (32 - q * BGBIT);
    OFF += 1u << (31 - L * BGBIT);
    constexpr int ROWS = 2 * L;

    for (uint32_t i = 0; i < n; i++) {
        __syncthreads();
        const uint32_t a = S.abar[i];
        if (a == 0)
            continue;
        uint32_t tmpA[16], tmpB[16];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int j = t + 64 * q;
            tmpA[q] = rot_read(S.acc[0], a, j) - S.acc[0][j] + OFF;
            tmpA[8 + q] = rot_read(S.acc[0], a, j + 512) - S.acc[0][j + 512] + OFF;
            tmpB[q] = rot_read(S.acc[1], a, j) - S.acc[1][j] + OFF;
            tmpB[8 + q] = rot_read(S.acc[1], a, j + 512) - S.acc[1][j + 512] + OFF;
        }
        const double2* bki = bkf + (size_t)i * ROWS * 2 * FFT_M;
        double2 oA[8], oB[8];
#pragma unroll 1
        for (int pr = 0; pr < L; pr++) {
            const int r0 = 2 * pr, r1 = 2 * pr + 1;
            const bool cb0 = r0 >= L, cb1 = r1 >= L;
            const int sh0 = 32 - ((r0 % L) + 1) * BGBIT, sh1 = 32 - ((r1 % L) + 1) * BGBIT;
            // comp-A BK slots of both rows in flight during the transforms
            const double2* row0 = bki + (size_t)r0 * 2 * FFT_M;
            const double2* row1 = bki + (size_t)r1 * 2 * FFT_M;
            double2 BA0[8], BA1[8];
#pragma unroll
            for (int q = 0; q < 8; q++) {
                BA0[q] = ld_stream(row0 + q * 64 + t);
                BA1[q] = ld_stream(row1 + q * 64 + t);
            }
            double2 x0[8], x1[8];
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const uint32_t lo0 = cb0 ? tmpB[q] : tmpA[q], hi0 = cb0 ? tmpB[8 + q] : tmpA[8 + q];
                const uint32_t lo1 = cb1 ? tmpB[q] : tmpA[q], hi1 = cb1 ? tmpB[8 + q] : tmpA[8 + q];
                const double2 twq = S.tws[t + 64 * q];
                x0[q] = cmul(make_double2((double)((int)((lo0 >> sh0) & MASK) - (int)HALF),
                                          (double)((int)((hi0 >> sh0) & MASK) - (int)HALF)), twq);
                x1[q] = cmul(make_double2((double)((int)((lo1 >> sh1) & MASK) - (int)HALF),
                                          (double)((int)((hi1 >> sh1) & MASK) - (int)HALF)), twq);
            }
            fft_forward2(x0, x1, tw, S.cross[0], S.cross[1], S.intra[0], S.intra[1], t, bar, wbar);
            // MAC (oracle row order r0 then r1) into the TMEM-resident accumulators
            if (pr > 0) {
                tmem_wait_st();
                tm_mac_load(tb, oA);
            } else {
#pragma unroll
                for (int q = 0; q < 8; q++)
                    oA[q] = make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int q = 0; q < 8; q++) {
                mac(oA[q], x0[q], BA0[q]);
                mac(oA[q], x1[q], BA1[q]);
            }
            if (pr + 1 < L)
                tm_mac_store(tb, oA);
            if (pr > 0)
                tm_mac_load(tb + 32, oB);
            else {
#pragma unroll
                for (int q = 0; q < 8; q++)
                    oB[q] = make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int q = 0; q < 8; q++) {
                mac(oB[q], x0[q], ld_stream(row0 + FFT_M + q * 64 + t));
                mac(oB[q], x1[q], ld_stream(row1 + FFT_M + q * 64 + t));
            }
            if (pr + 1 < L)
                tm_mac_store(tb + 32, oB);
        }
        // both inverse transforms together, round, accumulate into ACC
        fft_inverse2(oA, oB, tw, S.cross[0], S.cross[1], S.intra[0], S.intra[1], t, bar, wbar);
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int j = t + 64 * q;
            const double2 ut = untwist(S.tws[j]);
            const double2 wa = cmul(oA[q], ut);
            const double2 wb = cmul(oB[q], ut);
            S.acc[0][j] += (uint32_t)__double2ll_rn(wa.x);
            S.acc[0][j + 512] += (uint32_t)__double2ll_rn(wa.y);
            S.acc[1][j] += (uint32_t)__double2ll_rn(wb.x);
            S.acc[1][j + 512] += (uint32_t)__double2ll_rn(wb.y);
        }
    }
    __syncthreads();
    uint32_t* o = pool_N + (size_t)it.out * dp.N_stride;
    for (int j = t; j < 1024; j += 64)
        o[j] = j == 0 ? S.acc[0][0] : 0u - S.acc[0][1024 - j];
    if (t == 0)
        o[1024] = S.acc[1][0];
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (t < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;\n" ::"r"(S.tmem_slot));
}

}  // namespace lpb
