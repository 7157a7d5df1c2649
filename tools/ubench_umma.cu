// Microbenchmark: tcgen05.mma throughput per SM for the operand layouts the
// grid convolution can use (K-major, no swizzle vs 32/64/128-byte swizzle),
// kind::tf32 and kind::f16, M = 128, N = 32..256, one K step per instruction
// (K = 8 tf32 / 16 f16): one thread issues back-to-back MMAs into two TMEM
// accumulators, operands fixed in shared memory; cycles per MMA vs the dense
// peak (tf32: M N K / 1891 per SM cycle at 1.1 PFLOP/s).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/ubench_umma tools/ubench_umma.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout)
{
    return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)((lbo >> 4) & 0x3fffu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

// layout: 0 none (core matrices 8 rows x 16 B, SBO 128, LBO = rows x 16), 6 SW32 (rows of 32 B, SBO 256),
// 4 SW64 (rows of 64 B, SBO 512), 2 SW128 (rows of 128 B, SBO 1024)
template <int KIND>  // 0 tf32, 1 f16
__global__ void k_umma(long long* out, int N, int layout, int iters)
{
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long s_bar;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f800000u ^ (i * 2654435761u & 0x007fffffu);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    if (threadIdx.x == 0) {
        const uint32_t M = 128;
        uint32_t idesc;
        if (KIND == 0) idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((M >> 4) << 24);
        else idesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((M >> 4) << 24);
        const uint32_t a0 = base, b0 = base + 48 * 1024;
        uint32_t lbo_a, lbo_b, sbo;
        if (layout == 0) { lbo_a = M * 16; lbo_b = N * 16; sbo = 128; }
        else { lbo_a = lbo_b = 16; sbo = layout == 6 ? 256 : layout == 4 ? 512 : 1024; }
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            // vary the operand base over a few atoms like a streaming kernel does
            const uint32_t sa = a0 + (uint32_t)((it & 3) * 2048), sb = b0 + (uint32_t)((it & 1) * 8192);
            const uint64_t da = desc(sa, lbo_a, sbo, layout), db = desc(sb, lbo_b, sbo, layout);
            const uint32_t d = tmem + (uint32_t)((it & 1) * 256);
            if (KIND == 0)
                asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
                             ::"r"(d), "l"(da), "l"(db), "r"(idesc), "r"(it > 1 ? 1 : 0));
            else
                asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                             ::"r"(d), "l"(da), "l"(db), "r"(idesc), "r"(it > 1 ? 1 : 0));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(bar) : "memory");
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main()
{
    long long* d;
    cudaMalloc(&d, 1024 * sizeof(long long));
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(k_umma<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    cudaFuncSetAttribute(k_umma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int iters = 4096;
    for (int kind = 0; kind < 2; ++kind)
        for (int layout : {0, 6, 4, 2})
            for (int N : {32, 64, 128, 256}) {
                for (int rep = 0; rep < 2; ++rep) {
                    if (kind == 0) k_umma<0><<<sms, 128, 100 * 1024>>>(d, N, layout, iters);
                    else k_umma<1><<<sms, 128, 100 * 1024>>>(d, N, layout, iters);
                }
                cudaError_t e = cudaDeviceSynchronize();
                long long h[1024];
                cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
                double avg = 0;
                for (int i = 0; i < sms; ++i) avg += (double)h[i];
                avg /= sms;
                const double cyc = avg / iters;
                const double K = kind == 0 ? 8 : 16;
                const double peak_cyc = 128.0 * N * K / (kind == 0 ? 1891.0 : 3782.0);
                printf("%s layout %d N %3d: %7.1f cycles/MMA (dense peak %5.1f, %.2f of peak) %s\n", kind ? "f16 " : "tf32",
                       layout, N, cyc, peak_cyc, peak_cyc / cyc, e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
    return 0;
}
