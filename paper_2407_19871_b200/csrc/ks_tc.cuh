// ks_tc.cuh -- K2t: LWE key switching as an INT8 tensor-core contraction (tcgen05, sm_100a).
//
// Key switching (SURVEY §8(a'), the reference plug-in point gate_engine.hpp:117-123):
//   out = (0, b') - sum_{i<N, j<t} KSK[i][j][d_ij]          (d_ij in {0..3}; d = 0 adds nothing)
// where d_ij is the j-th 2-bit digit of a'_i + 2^15.  For a batch of ciphertexts this is a
// matrix product with a 0/1 matrix:
//   S[ct][col] = sum_{k = (i, j, d)} A[ct][k] * KSK[i][j][d][col],   A[ct][k] = [d_ij(ct) == d]
// over d = 1..3 only (d = 0 adds nothing): K = N t 3 = 24,576 (the order of k inside a
// stage is given at kt_slot_coef).  Every KSK word is split into its four
// bytes (column 4 col + b holds byte b), so both operands are unsigned 8-bit and the MMA
// runs as tcgen05.mma kind::i8 with int32 accumulators in tensor memory.  Each byte-column
// sum is at most N t * 255 = 2,088,960 < 2^31, so the accumulation is exact, and the epilogue
// rebuilds out = b' [col = n] - (S0 + S1 << 8 + S2 << 16 + S3 << 24) mod 2^32 -- bit-identical
// to the subtraction chain of K2 / the oracle (integer sums mod 2^32 are order-free).
//
// CTA = 2 x 128 ciphertexts (two M-halves sharing every B tile) x one N tile of 256
// byte-columns (64 output columns); 384 threads:
//   warp 0       B producer: one bulk async copy per stage of the pre-tiled KSK block
//   warp 1       MMA issuer (one thread): 2 halves x 3 K-steps of M128 N256 K32 per stage
//   warp 2       TMEM allocator (512 columns: two 128 x 256 int32 accumulators)
//   warps 4..11  A producers (thread = one ciphertext row of one half: one-hot bytes built
//                from the digit words, stored in the core-matrix layout), then the epilogue
//                (TMEM -> combine -> pool).  Warp w reads TMEM lane quarter w % 4.
// Operand layout in shared memory (K-major, SWIZZLE_NONE "interleaved" canonical form):
// a 16-byte K-chunk c of row r sits at c * LBO + r * 16, so eight consecutive rows form a
// contiguous 128-byte core matrix (SBO = 128).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lpb {

constexpr int KT_M = 128;             // rows (ciphertexts) per M-half
constexpr int KT_HALVES = 2;          // M-halves per CTA (share B)
constexpr int KT_N = 256;             // byte-columns per N tile (64 output columns)
constexpr int KT_KC = 96;             // K per stage (32 positions x digit values 1..3)
constexpr int KT_CHUNKS = KT_KC / 16; // 16-byte K chunks per row per stage
constexpr int KT_STAGES = 4;
constexpr int KT_A_BYTES = KT_M * KT_KC;         // 12 KB per half
constexpr int KT_B_BYTES = KT_N * KT_KC;         // 24 KB
constexpr int KT_STAGE_BYTES = KT_HALVES * KT_A_BYTES + KT_B_BYTES;  // 48 KB
constexpr int KT_BUILDERS = 8;  // A-producer / epilogue warps: one row each (4: 3.65 vs 3.12 ms)
constexpr int KT_HPT = KT_HALVES * 4 / KT_BUILDERS;     // M-halves per builder thread
constexpr int KT_THREADS = 128 + 32 * KT_BUILDERS;
// K2t's launch time is flat (~0.18 ms, one wave) up to ~3,800 ciphertexts; the split K2s
// grows linearly (0.10 / 0.13 ms at 128, 0.15 / 0.19 ms at 192, 0.83 ms at 1,024 for
// 80 / 128-bit; tools/ks_sweep.py): K2t from 192 ciphertexts on.
constexpr uint32_t KT_MIN_COUNT = 192;
constexpr size_t KT_SMEM = (size_t)KT_STAGES * KT_STAGE_BYTES + 1024;

__device__ __forceinline__ uint32_t kt_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void kt_mbar_init(uint64_t* b, uint32_t n)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(kt_smem(b)), "r"(n));
}
__device__ __forceinline__ void kt_mbar_arrive(uint64_t* b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(kt_smem(b)) : "memory");
}
__device__ __forceinline__ void kt_mbar_expect_tx(uint64_t* b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(kt_smem(b)),
                 "r"(bytes)
                 : "memory");
}
// bounded wait: a protocol error traps instead of hanging the GPU
__device__ __forceinline__ void kt_mbar_wait(uint64_t* b, uint32_t phase)
{
    uint32_t done = 0;
    for (uint32_t it = 0; !done; it++) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(kt_smem(b)), "r"(phase)
            : "memory");
        if (it > (1u << 24))
            __trap();
    }
}
__device__ __forceinline__ void kt_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile(
        "{\n\t.reg .b64 pol;\n\t"
        "createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], pol;\n\t}\n" ::"r"(kt_smem(dst)),
        "l"(src), "r"(bytes), "r"(kt_smem(bar))
        : "memory");
}
// UMMA shared-memory descriptor: K-major, no swizzle, version 1 (sm_100)
__device__ __forceinline__ uint64_t kt_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // version
    return d;               // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}
// instruction descriptor: D s32, A u8, B u8, both K-major, N = 256, M = 128
constexpr uint32_t KT_IDESC = (2u << 4) | ((uint32_t)(KT_N >> 3) << 17) | ((uint32_t)(KT_M >> 4) << 24);

__device__ __forceinline__ void kt_mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(KT_IDESC), "r"(acc));
}
__device__ __forceinline__ void kt_commit(uint64_t* bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     kt_smem(bar))
                 : "memory");
}
__device__ __forceinline__ void kt_tmem_ld64(uint32_t addr, uint32_t (&v)[64])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,"
        "%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,"
        "%56,%57,%58,%59,%60,%61,%62,%63}, [%64];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]),
          "=r"(v[32]), "=r"(v[33]), "=r"(v[34]), "=r"(v[35]), "=r"(v[36]), "=r"(v[37]),
          "=r"(v[38]), "=r"(v[39]), "=r"(v[40]), "=r"(v[41]), "=r"(v[42]), "=r"(v[43]),
          "=r"(v[44]), "=r"(v[45]), "=r"(v[46]), "=r"(v[47]), "=r"(v[48]), "=r"(v[49]),
          "=r"(v[50]), "=r"(v[51]), "=r"(v[52]), "=r"(v[53]), "=r"(v[54]), "=r"(v[55]),
          "=r"(v[56]), "=r"(v[57]), "=r"(v[58]), "=r"(v[59]), "=r"(v[60]), "=r"(v[61]),
          "=r"(v[62]), "=r"(v[63])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// K order inside a stage (96 = 3 digit values x 8 digit positions x 4 coefficients), chosen
// so the A rows are cheap to build: k = 32 (d - 1) + 4 j + s, where digit position j of
// coefficient i = 4 kc + KT_SLOT_COEF[s] has value d.
__host__ __device__ constexpr uint32_t kt_slot_coef(uint32_t s) { return (0x3120u >> (4 * s)) & 15u; }

// KSK -> the tiled byte layout the MMA consumes, once per upload.  Block (nt, kc) (24 KB,
// contiguous) = [c < 6][n < 256][16 bytes]: byte b of chunk c of byte-column n is K index
// k = 16c + b of stage kc (order above); it holds byte (n % 4) of KSK[i][j][d-1][n / 4]
// (0 for a padding column).
__global__ void k_ksk_to_tc(DevParams dp, const uint32_t* __restrict__ ksk, uint32_t n_tiles,
                            uint4* __restrict__ out)
{
    const uint32_t kc_count = dp.N * dp.t * 3 / KT_KC;
    const uint64_t total = (uint64_t)n_tiles * kc_count * KT_CHUNKS * KT_N;  // 16-byte chunks
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t nl = (uint32_t)(e % KT_N);
        const uint32_t c = (uint32_t)((e / KT_N) % KT_CHUNKS);
        const uint64_t blk = e / (KT_N * KT_CHUNKS);
        const uint32_t kc = (uint32_t)(blk % kc_count), nt = (uint32_t)(blk / kc_count);
        const uint32_t n = nt * KT_N + nl, col = n / 4, byte = n % 4;
        uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
        for (int b = 0; b < 16; b++) {
            const uint32_t kk = 16 * c + b, d = kk / 32, j = (kk % 32) / 4;
            const uint32_t i = 4 * kc + kt_slot_coef(kk % 4);
            uint32_t v = 0;
            if (col <= dp.n)
                v = (ksk[((size_t)(i * dp.t + j) * 3 + d) * dp.n_stride + col] >> (8 * byte)) & 255u;
            w[b / 4] |= v << (8 * (b % 4));
        }
        out[e] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

__global__ void __launch_bounds__(KT_THREADS, 1)
    k_keyswitch_tc(DevParams dp, const KsItem* __restrict__ items, uint32_t count,
                   const uint32_t* __restrict__ pool_N, uint32_t* __restrict__ pool_n,
                   const uint4* __restrict__ kskt)
{
    extern __shared__ __align__(1024) uint8_t kt_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)kt_raw + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t full_bar[KT_STAGES], empty_bar[KT_STAGES], acc_bar;
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nt = blockIdx.x;  // adjacent CTAs share one M tile's inputs (L2 hits)
    const uint32_t ct0 = blockIdx.y * (KT_M * KT_HALVES);
    const uint32_t kc_count = dp.N * dp.t * 3 / KT_KC;
    const uint32_t prec = 1u << (32 - (1 + dp.basebit * dp.t));

    if (threadIdx.x == 0) {
        for (int s = 0; s < KT_STAGES; s++) {
            kt_mbar_init(&full_bar[s], 1 + KT_BUILDERS);  // B producer (expect_tx) + A-producer warps
            kt_mbar_init(&empty_bar[s], 1);     // tcgen05.commit
        }
        kt_mbar_init(&acc_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
            kt_smem(&tmem_base_sh)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base_sh;

    auto stage_a = [&](int s, int h) { return smem + (size_t)s * KT_STAGE_BYTES + h * KT_A_BYTES; };
    auto stage_b = [&](int s) { return smem + (size_t)s * KT_STAGE_BYTES + KT_HALVES * KT_A_BYTES; };

    if (warp == 0) {
        // ---- B producer
        if (lane == 0) {
            const uint8_t* src = reinterpret_cast<const uint8_t*>(kskt) + (size_t)nt * kc_count * KT_B_BYTES;
            for (uint32_t kc = 0; kc < kc_count; kc++) {
                const int s = kc % KT_STAGES;
                const uint32_t ph = (kc / KT_STAGES) & 1u;
                if (kc >= KT_STAGES)
                    kt_mbar_wait(&empty_bar[s], ph ^ 1u);
                kt_mbar_expect_tx(&full_bar[s], KT_B_BYTES);
                kt_bulk_g2s(stage_b(s), src + (size_t)kc * KT_B_BYTES, KT_B_BYTES, &full_bar[s]);
            }
        }
    } else if (warp == 1) {
        // ---- MMA issuer
        if (lane == 0) {
            for (uint32_t kc = 0; kc < kc_count; kc++) {
                const int s = kc % KT_STAGES;
                kt_mbar_wait(&full_bar[s], (kc / KT_STAGES) & 1u);
                asm volatile("tcgen05.fence::after_thread_sync;\n");
                const uint32_t b0 = kt_smem(stage_b(s));
#pragma unroll
                for (int h = 0; h < KT_HALVES; h++) {
                    const uint32_t a0 = kt_smem(stage_a(s, h));
#pragma unroll
                    for (int kk = 0; kk < KT_KC / 32; kk++) {
                        const uint64_t ad = kt_desc(a0 + kk * 2 * (KT_M * 16), KT_M * 16, 128);
                        const uint64_t bd = kt_desc(b0 + kk * 2 * (KT_N * 16), KT_N * 16, 128);
                        kt_mma(tmem + h * KT_N, ad, bd, (kc | kk) != 0);
                    }
                }
                kt_commit(&empty_bar[s]);  // stage free once these MMAs have read it
            }
            kt_commit(&acc_bar);  // accumulators complete
        }
    } else if (warp >= 4) {
        // ---- A producers: thread r builds row r of M-halves h0 .. h0 + KT_HPT - 1
        // (ciphertexts ct0 + h*128 + r); warp w reads TMEM lane quarter w % 4 in the epilogue
        const int r = (warp & 3) * 32 + lane;
        const int h0 = (warp - 4) / 4 * KT_HPT;
        const uint32_t* a0p[KT_HPT];
        const uint32_t* a1p[KT_HPT];
#pragma unroll
        for (int h = 0; h < KT_HPT; h++) {
            const uint32_t g = ct0 + (h0 + h) * KT_M + r;
            a0p[h] = a1p[h] = nullptr;
            if (g < count) {
                const KsItem it = items[g];
                LPB_ASSERT(it.in0 < dp.scratch_slots && it.out < dp.pool_slots &&
                           (it.in1 == SLOT_NONE || it.in1 < dp.scratch_slots));
                a0p[h] = pool_N + (size_t)it.in0 * dp.N_stride;
                a1p[h] = it.in1 != SLOT_NONE ? pool_N + (size_t)it.in1 * dp.N_stride : nullptr;
            }
        }
        // digit words for two stages (8 coefficients = one 32-byte sector per input row)
        // are loaded one stage pair ahead, so the L2 latency overlaps the previous pair
        uint4 cur[KT_HPT][2][2], nxt[KT_HPT][2][2];  // [half][input][stage of pair]
        auto load_pair = [&](uint32_t kp, uint4 (&d)[KT_HPT][2][2]) {
#pragma unroll
            for (int h = 0; h < KT_HPT; h++)
#pragma unroll
                for (int e = 0; e < 2; e++) {
                    d[h][0][e] = a0p[h] ? __ldg(reinterpret_cast<const uint4*>(a0p[h] + 8 * kp + 4 * e))
                                        : make_uint4(0, 0, 0, 0);
                    d[h][1][e] = a1p[h] ? __ldg(reinterpret_cast<const uint4*>(a1p[h] + 8 * kp + 4 * e))
                                        : make_uint4(0, 0, 0, 0);
                }
        };
        load_pair(0, cur);
        for (uint32_t kp = 0; kp < kc_count / 2; kp++) {
            if (kp + 1 < kc_count / 2)
                load_pair(kp + 1, nxt);
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const uint32_t kc = 2 * kp + e;
                const int s = kc % KT_STAGES;
                if (kc >= KT_STAGES)
                    kt_mbar_wait(&empty_bar[s], ((kc / KT_STAGES) & 1u) ^ 1u);
                // this stage covers coefficients i = 4 kc .. 4 kc + 3 (t = 8 positions each)
#pragma unroll
                for (int h = 0; h < KT_HPT; h++) {
                    const uint4 w0 = cur[h][0][e], w1 = cur[h][1][e];
                    const uint32_t wd[4] = {(w0.x + w1.x + prec) >> 16, (w0.y + w1.y + prec) >> 16,
                                            (w0.z + w1.z + prec) >> 16, (w0.w + w1.w + prec) >> 16};
                    uint8_t* dst = stage_a(s, h0 + h) + r * 16;
                    const uint32_t live = a0p[h] != nullptr ? 0x01010101u : 0u;
                    // word (d, j): byte s = [digit j of coefficient kt_slot_coef(s) == d]
                    const uint32_t P = wd[0] | (wd[1] << 16), Q = wd[2] | (wd[3] << 16);
                    uint32_t wv[24];
#pragma unroll
                    for (int j = 0; j < 8; j++) {
                        // bytes (c0, c2, c1, c3) of digit j
                        const uint32_t dj = ((P >> (14 - 2 * j)) & 0x00030003u) |
                                            (((Q >> (14 - 2 * j)) & 0x00030003u) << 8);
#pragma unroll
                        for (int d = 1; d <= 3; d++) {
                            const uint32_t y = dj ^ (0x01010101u * (uint32_t)d);  // 0 where equal
                            wv[8 * (d - 1) + j] = ~(y | (y >> 1)) & live;
                        }
                    }
#pragma unroll
                    for (int c = 0; c < KT_CHUNKS; c++)
                        *reinterpret_cast<uint4*>(dst + c * (KT_M * 16)) =
                            make_uint4(wv[4 * c], wv[4 * c + 1], wv[4 * c + 2], wv[4 * c + 3]);
                }
                asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                __syncwarp();
                if (lane == 0)
                    kt_mbar_arrive(&full_bar[s]);
            }
#pragma unroll
            for (int h = 0; h < KT_HPT; h++)
#pragma unroll
                for (int i = 0; i < 2; i++)
#pragma unroll
                    for (int e = 0; e < 2; e++)
                        cur[h][i][e] = nxt[h][i][e];
        }
        // ---- epilogue: TMEM lane quarter (warp & 3) -> rows r; 64 output columns per half
        kt_mbar_wait(&acc_bar, 0);
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        const uint32_t lane_addr = (uint32_t)((warp & 3) * 32) << 16;
#pragma unroll 1
        for (int h = h0; h < h0 + KT_HPT; h++) {
            const uint32_t g = ct0 + h * KT_M + r;
            const bool live = g < count;
            KsItem it{};
            uint32_t body = 0;
            if (live) {
                it = items[g];
                body = pool_N[(size_t)it.in0 * dp.N_stride + dp.N] + it.off;
                if (it.in1 != SLOT_NONE)
                    body += pool_N[(size_t)it.in1 * dp.N_stride + dp.N];
            }
#pragma unroll 1
            for (int q = 0; q < 4; q++) {  // 64 byte-columns = 16 output columns per load
                uint32_t v[64];
                kt_tmem_ld64(tmem + lane_addr + h * KT_N + 64 * q, v);
                if (!live)
                    continue;
                uint32_t o[16];
#pragma unroll
                for (int c = 0; c < 16; c++) {
                    const uint32_t col = nt * (KT_N / 4) + 16 * q + c;
                    const uint32_t sum = v[4 * c] + (v[4 * c + 1] << 8) + (v[4 * c + 2] << 16) +
                                         (v[4 * c + 3] << 24);
                    o[c] = (col == dp.n ? body : 0u) - sum;
                }
                const uint32_t col0 = nt * (KT_N / 4) + 16 * q;
                uint32_t* dstp = pool_n + (size_t)it.out * dp.n_stride + col0;
#pragma unroll
                for (int c = 0; c < 16; c += 4)
                    if (col0 + c < dp.n_stride)
                        *reinterpret_cast<uint4*>(dstp + c) = make_uint4(o[c], o[c + 1], o[c + 2], o[c + 3]);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp == 2)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

}  // namespace lpb
