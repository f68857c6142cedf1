// br_cluster.cuh -- K1x: latency blind rotation on a cluster of 2l CTAs per ciphertext.
//
// For levels far smaller than the GPU (cfg1: one query, a few to a few dozen bootstraps per
// level) a blind rotation is latency-bound: K1l puts all 2l digit transforms, the MAC and
// both inverse transforms of a CMux step on one SM.  Here the 2l digit rows of a step run
// on 2l SMs: CTA rank r = (c, p) (c = r / l, p = r % l) owns ACC component c and
//   1. forms digit p of (X^a - 1) ACC_c and its forward transform (64 threads);
//   2. stores the spectrum into slot [r] of every cluster CTA's F tile (DSMEM);
//   3. after one cluster barrier, runs the MAC for output component c over all 2l rows in
//      the oracle's row order (same fma chain as K1/K1l: bit-exact), with the 2l BK rows
//      of component c bulk-copied into shared memory one executed step ahead;
//   4. inverse-transforms output c and updates its copy of ACC_c.
// The l CTAs of a component compute the same MAC + inverse redundantly, so ACC_c never
// crosses SMs and one cluster barrier per step suffices: F is double-buffered by step
// parity, and a CTA writes F[parity] of step k+2 only after the barrier of step k+1, which
// every peer reaches after finishing the MAC of step k.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"
#include "ks_tc.cuh"

namespace lpb {

template <int L>
struct ClSmem {
    double2 F[2][2 * L][FFT_M];  // [step parity][row][slot q*64+t]: every row's spectrum
    double2 B[2][2 * L][FFT_M];  // [buffer][row]: BK_i row, this CTA's output component
    double2 tiles[2][XTILE];     // cross-warp / intra-warp exchange tiles
    uint32_t acc[1024];          // ACC component c
    uint16_t abar[MAX_N + 1];
    uint64_t bk_bar[2];
};
template <int L>
constexpr size_t kClSmemBytes = sizeof(ClSmem<L>) + 128;

__device__ __forceinline__ uint32_t cl_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cl_map(const void* p, uint32_t rank)
{
    uint32_t out;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(out) : "r"(kt_smem(p)), "r"(rank));
    return out;
}
__device__ __forceinline__ void cl_st(uint32_t addr, double2 v)
{
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};\n" ::"r"(addr), "d"(v.x), "d"(v.y)
                 : "memory");
}
__device__ __forceinline__ void cl_sync()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::
                     : "memory");
}

template <int L, int BGBIT>
__global__ void __launch_bounds__(64, 1)
    k_blind_rotate_cl(DevParams dp, const BrItem* __restrict__ items,
                      const uint32_t* __restrict__ pool_n, uint32_t* __restrict__ pool_N,
                      const double2* __restrict__ bkf, FftTabs tb, uint32_t mu)
{
    constexpr int R = 2 * L;
    extern __shared__ uint8_t smem_cl_raw[];
    ClSmem<L>& S = *reinterpret_cast<ClSmem<L>*>(((uintptr_t)smem_cl_raw + 127) & ~(uintptr_t)127);
    const uint32_t rank = cl_rank();
    const int c = (int)rank / L, p = (int)rank % L;
    const int t = threadIdx.x;
    const BrItem it = items[blockIdx.x / R];
    const uint32_t n = dp.n;
    LPB_ASSERT(it.in0 < dp.pool_slots && it.out < dp.scratch_slots && n <= MAX_N);
    LPB_ASSERT((it.in1 == SLOT_NONE || it.in1 < dp.pool_slots) &&
               (it.in2 == SLOT_NONE || it.in2 < dp.pool_slots));

    // ---- prologue: gate linear form + mod switch (as K1), ACC_c = test vector component c
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
    if (t == 0) {
        kt_mbar_init(&S.bk_bar[0], 1);
        kt_mbar_init(&S.bk_bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    {
        const uint32_t e = (2048u - S.abar[n]) & 2047u;
        for (int j = t; j < 1024; j += 64) {
            const uint32_t idx = (uint32_t)(j - (int)e) & 2047u;
            S.acc[j] = c == 0 ? 0u : (idx < 1024u ? mu : 0u - mu);
        }
    }
    uint32_t fpeer[R];  // F[0][0][0] of every cluster CTA
#pragma unroll
    for (int q = 0; q < R; q++)
        fpeer[q] = cl_map(&S.F[0][0][0], (uint32_t)q);

    const FwdTw tw = load_fwd_tw(tb.fwd, t);
    const double2 twt = tb.tw[t];
    auto bar = [] {
        lpb_jitter();
        __syncthreads();
    };
    auto wbar = [] {
        lpb_jitter();
        __syncwarp();
    };
    constexpr uint32_t HALF = 1u << (BGBIT - 1);
    constexpr uint32_t MASK = (1u << BGBIT) - 1;
    uint32_t OFF = 0;
#pragma unroll
    for (int q = 1; q <= L; q++)
        OFF += HALF << (32 - q * BGBIT);
    OFF += 1u << (31 - L * BGBIT);
    const int sh = 32 - (p + 1) * BGBIT;

    auto next_step = [&](uint32_t i) {
        while (i < n && S.abar[i] == 0)
            i++;
        return i;
    };
    // BK_i rows r = 0..R-1 of output component c -> S.B[buf] (8 KB bulk copies)
    auto issue_bk = [&](uint32_t i, int buf) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        kt_mbar_expect_tx(&S.bk_bar[buf], (uint32_t)(R * FFT_M * sizeof(double2)));
#pragma unroll 1
        for (int r = 0; r < R; r++)
            kt_bulk_g2s(&S.B[buf][r][0], bkf + ((size_t)i * R + r) * 2 * FFT_M + (size_t)c * FFT_M,
                        (uint32_t)(FFT_M * sizeof(double2)), &S.bk_bar[buf]);
    };

    __syncthreads();
    cl_sync();  // every peer's shared memory is live before the first DSMEM store
    uint32_t i = next_step(0);
    if (t == 0 && i < n)
        issue_bk(i, 0);
    for (uint32_t k = 0; i < n; k++) {
        const uint32_t a = S.abar[i];
        const int buf = (int)(k & 1u);
        const uint32_t inext = next_step(i + 1);
        if (t == 0 && inext < n)  // buffer buf^1 was last read by the MAC of step k-1
            issue_bk(inext, buf ^ 1);
        // ---- digit p of (X^a - 1) ACC_c -> forward transform
        double2 x[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int j = t + 64 * q;
            const uint32_t lo = rot_read(S.acc, a, j) - S.acc[j] + OFF;
            const uint32_t hi = rot_read(S.acc, a, j + 512) - S.acc[j + 512] + OFF;
            const int dlo = (int)((lo >> sh) & MASK) - (int)HALF;
            const int dhi = (int)((hi >> sh) & MASK) - (int)HALF;
            x[q] = make_double2((double)dlo, (double)dhi);
        }
        fft_forward(x, tw, S.tiles[0], S.tiles[1], t, bar, wbar);
        // ---- spectrum of row `rank` into F[parity][rank] of every cluster CTA
        {
            const uint32_t off =
                (uint32_t)((((size_t)buf * R + rank) * FFT_M + t) * sizeof(double2));
#pragma unroll
            for (int q2 = 0; q2 < R; q2++)
#pragma unroll
                for (int q = 0; q < 8; q++)
                    cl_st(fpeer[q2] + off + (uint32_t)(q * 64 * sizeof(double2)), x[q]);
        }
        cl_sync();
        // ---- MAC for output c, rows 0..R-1 in order (the oracle's chain)
        kt_mbar_wait(&S.bk_bar[buf], (k >> 1) & 1u);
        double2 o[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            o[q] = make_double2(0.0, 0.0);
#pragma unroll
            for (int r = 0; r < R; r++)
                mac(o[q], S.F[buf][r][q * 64 + t], S.B[buf][r][q * 64 + t]);
        }
        {
            const InvTw itw = load_inv_tw(tb.inv, t);
            fft_inverse(o, itw, S.tiles[0], S.tiles[1], t, bar, wbar);
        }
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int j = t + 64 * q;
            const double2 w = cmul(o[q], untwist(twt, q));
            S.acc[j] += (uint32_t)__double2ll_rn(w.x);
            S.acc[j + 512] += (uint32_t)__double2ll_rn(w.y);
        }
        __syncthreads();
        i = inext;
    }
    // ---- sample extraction: a' from component 0 (rank 0), b' from component 1 (rank L)
    uint32_t* out = pool_N + (size_t)it.out * dp.N_stride;
    if (rank == 0)
        for (int j = t; j < 1024; j += 64)
            out[j] = j == 0 ? S.acc[0] : 0u - S.acc[1024 - j];
    if (rank == (uint32_t)L && t == 0)
        out[1024] = S.acc[0];
    cl_sync();  // no CTA leaves while a peer could still address its shared memory
}

}  // namespace lpb
