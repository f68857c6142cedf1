// microbench.cu -- B200 data-path throughput probes that shape the blind-rotate
// kernel design: TMEM (tcgen05.ld/st 32x32b) vs shared memory (LDS/STS.128) vs
// warp shuffles, per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_tmem(uint32_t* out, int iters, int do_store)
{
    __shared__ uint32_t taddr;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"l"((uint64_t)__cvta_generic_to_shared(&taddr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t base = taddr + (((uint32_t)(warp & 3) * 32) << 16);
    uint32_t a0 = threadIdx.x, a1 = 1, a2 = 2, a3 = 3, a4 = 4, a5 = 5, a6 = 6, a7 = 7;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(base), "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(a4), "r"(a5), "r"(a6), "r"(a7));
    asm volatile("tcgen05.wait::st.sync.aligned;\n");
    uint32_t acc = 0;
    for (int i = 0; i < iters; i++) {
        const uint32_t col = base + ((i & 7) * 8);
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                     : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3), "=r"(a4), "=r"(a5), "=r"(a6), "=r"(a7) : "r"(col));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        acc += a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
        if (do_store) {
            a0 += 1;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(col), "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(a4), "r"(a5), "r"(a6), "r"(a7));
        }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n");
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;\n" ::"r"(taddr));
}

__global__ void k_smem(uint32_t* out, int iters)
{
    __shared__ uint4 buf[1024];
    buf[threadIdx.x] = make_uint4(threadIdx.x, 1, 2, 3);
    __syncthreads();
    uint32_t acc = 0;
    for (int i = 0; i < iters; i++) {
        uint4 v = buf[(threadIdx.x + i * 32) & 1023];
        acc += v.x ^ v.y ^ v.z ^ v.w;
        buf[(threadIdx.x + i * 64 + 7) & 1023] = make_uint4(acc, v.x, v.y, i);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_shfl(uint32_t* out, int iters)
{
    uint32_t a = threadIdx.x, b = 1, c = 2, d = 3;
    for (int i = 0; i < iters; i++) {
        a = __shfl_xor_sync(0xffffffffu, a, 1) + 1;
        b = __shfl_xor_sync(0xffffffffu, b, 2) + 1;
        c = __shfl_xor_sync(0xffffffffu, c, 4) + 1;
        d = __shfl_xor_sync(0xffffffffu, d, 8) + 1;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a ^ b ^ c ^ d;
}

int main()
{
    int sms = 0, clk = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    uint32_t* out;
    CK(cudaMalloc(&out, 64 << 20));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 1 << 14;
    auto report = [&](const char* what, double bytes, float ms) {
        const double cyc = ms * 1e-3 * clk * 1e3;
        printf("%-34s %8.3f ms  %8.1f B/clk/SM\n", what, ms, bytes / cyc / sms);
    };
    for (int ctas = 1; ctas <= 4; ctas *= 2)
        for (int st = 0; st <= 1; st++) {
            k_tmem<<<sms * ctas, 128>>>(out, 64, st);
            CK(cudaDeviceSynchronize());
            cudaEventRecord(e0);
            k_tmem<<<sms * ctas, 128>>>(out, iters, st);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            char name[64];
            snprintf(name, 64, "tmem ld%s x8, %d CTA/SM", st ? "+st" : "", ctas);
            report(name, (double)sms * ctas * 128 * iters * 32.0 * (st ? 2 : 1), ms);
        }
    for (int w = 4; w <= 16; w *= 2) {
        k_smem<<<sms, 32 * w>>>(out, 64);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        k_smem<<<sms, 32 * w>>>(out, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        char name[64];
        snprintf(name, 64, "smem lds+sts.128, %d warps/SM", w);
        report(name, (double)sms * 32 * w * iters * 32.0, ms);
    }
    for (int w = 4; w <= 16; w *= 2) {
        k_shfl<<<sms, 32 * w>>>(out, 64);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        k_shfl<<<sms, 32 * w>>>(out, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        char name[64];
        snprintf(name, 64, "shfl.b32 (4 per iter), %d warps/SM", w);
        report(name, (double)sms * 32 * w * iters * 16.0, ms);
    }
    return 0;
}
