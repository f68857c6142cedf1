// br_lat2.cuh -- latency blind rotation on a 2-CTA cluster per ciphertext (K1c, sm_100a).
//
// For small levels (cfg1-like single queries) a blind rotation is one ciphertext per SM
// and latency-bound: per CMux step the SM runs all 2l digit transforms and streams the
// whole BK_i.  Here a thread-block cluster of two CTAs shares the work by ACC component:
// CTA c owns ACC_c, computes the l digit transforms of (X^a - 1) ACC_c and loads only
// BK rows c*l .. c*l+l-1.  The external product keeps the oracle's per-slot MAC chain
// over rows 0 .. 2l-1 (bit-exact): CTA 0 runs rows 0..l-1 for both outputs and stores
// the partial sums into CTA 1's shared memory (DSMEM); CTA 1 continues rows l..2l-1,
// keeps output B and stores output A back into CTA 0; each CTA then inverse-transforms
// its own component.  Exchange buffers alternate by step parity, so two cluster barriers
// per step suffice.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft.cuh"
#include "kernels.cuh"

namespace lpb {

template <int L>
struct Lat2Smem {
    uint32_t acc[1024];                 // this CTA's ACC component
    double2 tws[FFT_M];
    double2 F[L][FFT_M];                // this CTA's digit spectra, slot layout [q*64 + t]
    double2 P[2][2][FFT_M];             // [step parity][output][slot]: partials / results
    double2 tiles[L][2][XTILE];
    uint16_t abar[MAX_N + 1];
};

template <int L, int BGBIT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64 * L, 1)
    k_blind_rotate_lat2(DevParams dp, const BrItem* __restrict__ items,
                        const uint32_t* __restrict__ pool_n, uint32_t* __restrict__ pool_N,
                        const double2* __restrict__ bkf, const double2* __restrict__ W,
                        const double2* __restrict__ TW, uint32_t mu)
{
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) uint8_t smem_l2[];
    Lat2Smem<L>& S = *reinterpret_cast<Lat2Smem<L>*>(smem_l2);
    const int comp = (int)cluster.block_rank();  // 0: component A, 1: component B
    const int g = threadIdx.x >> 6, t = threadIdx.x & 63;
    const BrItem it = items[blockIdx.x >> 1];
    const uint32_t n = dp.n;
    for (int j = threadIdx.x; j < FFT_M; j += blockDim.x)
        S.tws[j] = TW[j];
    {
        const uint32_t* a0 = pool_n + (size_t)it.in0 * dp.n_stride;
        const uint32_t* a1 = it.in1 != SLOT_NONE ? pool_n + (size_t)it.in1 * dp.n_stride : nullptr;
        const uint32_t* a2 = it.in2 != SLOT_NONE ? pool_n + (size_t)it.in2 * dp.n_stride : nullptr;
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
            const uint32_t idx = (uint32_t)(j - (int)e) & 2047u;
            S.acc[j] = comp == 0 ? 0u : (idx < 1024u ? mu : 0u - mu);
        }
    }
    const Twiddles tw = load_twiddles(W, t);
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
    const int sh = 32 - (g + 1) * BGBIT;
    // MAC slots of this thread: q = g + L*k (k < P), both outputs, this CTA's l rows
    constexpr int P = (8 + L - 1) / L;
    // the peer CTA's exchange buffers
    double2* peerP = cluster.map_shared_rank(&S.P[0][0][0], comp ^ 1);
    uint32_t par = 0;

    for (uint32_t i = 0; i < n; i++) {
        __syncthreads();
        const uint32_t a = S.abar[i];
        if (a == 0)
            continue;
        double2 bkv[L][2][P];
        {
            const double2* bki = bkf + (size_t)i * ROWS * 2 * FFT_M;
#pragma unroll
            for (int r = 0; r < L; r++)
#pragma unroll
                for (int o = 0; o < 2; o++)
#pragma unroll
                    for (int k = 0; k < P; k++) {
                        const int q = g + L * k;
                        if (q < 8)
                            bkv[r][o][k] = ld_stream(bki + ((size_t)(comp * L + r) * 2 + o) * FFT_M +
                                                     q * 64 + t);
                    }
        }
        {
            double2 x[8];
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const int j = t + 64 * q;
                const uint32_t lo = rot_read(S.acc, a, j) - S.acc[j] + OFF;
                const uint32_t hi = rot_read(S.acc, a, j + 512) - S.acc[j + 512] + OFF;
                const int dlo = (int)((lo >> sh) & MASK) - (int)HALF;
                const int dhi = (int)((hi >> sh) & MASK) - (int)HALF;
                x[q] = cmul(make_double2((double)dlo, (double)dhi), S.tws[j]);
            }
            fft_forward(x, tw, S.tiles[g][0], S.tiles[g][1], t, bar, wbar);
#pragma unroll
            for (int q = 0; q < 8; q++)
                S.F[g][q * 64 + t] = x[q];
        }
        __syncthreads();
        if (comp == 0) {
            // rows 0..l-1 from zero, both outputs -> CTA 1
#pragma unroll
            for (int k = 0; k < P; k++) {
                const int q = g + L * k;
                if (q < 8) {
#pragma unroll
                    for (int o = 0; o < 2; o++) {
                        double2 acc2 = make_double2(0.0, 0.0);
#pragma unroll
                        for (int r = 0; r < L; r++)
                            mac(acc2, S.F[r][q * 64 + t], bkv[r][o][k]);
                        peerP[(par * 2 + o) * FFT_M + q * 64 + t] = acc2;
                    }
                }
            }
        }
        cluster.sync();
        if (comp == 1) {
            // continue both chains with rows l..2l-1; keep B, return A to CTA 0
#pragma unroll
            for (int k = 0; k < P; k++) {
                const int q = g + L * k;
                if (q < 8) {
#pragma unroll
                    for (int o = 0; o < 2; o++) {
                        double2 acc2 = S.P[par][o][q * 64 + t];
#pragma unroll
                        for (int r = 0; r < L; r++)
                            mac(acc2, S.F[r][q * 64 + t], bkv[r][o][k]);
                        if (o == 0)
                            peerP[(par * 2 + 0) * FFT_M + q * 64 + t] = acc2;
                        else
                            S.P[par][1][q * 64 + t] = acc2;
                    }
                }
            }
        }
        cluster.sync();
        if (g == 0) {
            double2 o[8];
#pragma unroll
            for (int q = 0; q < 8; q++)
                o[q] = S.P[par][comp][q * 64 + t];
            fft_inverse(o, tw, S.tiles[0][0], S.tiles[0][1], t, bar, wbar);
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const int j = t + 64 * q;
                const double2 w = cmul(o[q], untwist(S.tws[j]));
                S.acc[j] += (uint32_t)__double2ll_rn(w.x);
                S.acc[j + 512] += (uint32_t)__double2ll_rn(w.y);
            }
        }
        par ^= 1u;
    }
    __syncthreads();
    uint32_t* out = pool_N + (size_t)it.out * dp.N_stride;
    if (comp == 0) {
        for (int j = threadIdx.x; j < 1024; j += blockDim.x)
            out[j] = j == 0 ? S.acc[0] : 0u - S.acc[1024 - j];
    } else if (threadIdx.x == 0) {
        out[1024] = S.acc[0];
    }
    cluster.sync();  // keep both CTAs' shared memory alive until the peer is done with it
}

}  // namespace lpb
