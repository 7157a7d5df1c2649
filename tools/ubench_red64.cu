// Microbenchmark: shared-memory reductions without return (red.shared.add)
// of 32-bit vs 64-bit words, consecutive lanes on consecutive words (the
// k_direct access pattern: one warp adds a profile's taps to one tile row).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int BITS>
__global__ void k_red(int* out, int iters) {
  extern __shared__ __align__(16) unsigned char sm[];
  int* s = reinterpret_cast<int*>(sm);
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) s[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t base = (uint32_t)__cvta_generic_to_shared(s);
  uint32_t off = (warp * 1237u) & 4095u;
  for (int it = 0; it < iters; ++it) {
    if (BITS == 32) {
      const uint32_t a = base + 4u * ((off + lane) & 16383u);
      asm volatile("red.shared.add.s32 [%0], %1;" :: "r"(a), "r"(it) : "memory");
      asm volatile("red.shared.add.s32 [%0+128], %1;" :: "r"(a), "r"(it) : "memory");
    } else {
      const uint32_t a = base + 8u * ((off + lane) & 8191u);
      asm volatile("red.shared.add.u64 [%0], %1;" :: "r"(a), "l"((unsigned long long)it * 0x100000001ull) : "memory");
    }
    off = (off + 160u) & 4095u;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[5];
}
int main() {
  int* d; cudaMalloc(&d, 4096 * 4);
  cudaFuncSetAttribute(k_red<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(k_red<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 8192, threads = 640, blocks = sms * 2;
  for (int rep = 0; rep < 3; ++rep)
    for (int bits : {32, 64}) {
      cudaEventRecord(a);
      if (bits == 32) k_red<32><<<blocks, threads, 100000>>>(d, iters);
      else k_red<64><<<blocks, threads, 100000>>>(d, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double taps = (double)blocks * threads * iters * 2;  // two 32-bit taps per lane-iteration either way
      if (rep) printf("red.shared %d-bit: %.3f ms, %.2f G taps/s, %.2f taps/clk/SM @1.965GHz\n", bits, ms, taps / ms / 1e6, taps / (ms * 1e-3) / sms / 1.965e9);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
