// Microbenchmark: shared-memory int32 atomicAdd (ATOMS.ADD) throughput with
// spread addresses vs plain LDS/STS read-modify-write, on one SM-wide sweep.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_atoms(int* out, int iters, int stride) {
  extern __shared__ int s[];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) s[i] = 0;
  __syncthreads();
  unsigned idx = (threadIdx.x * stride) & 16383;
  for (int it = 0; it < iters; ++it) {
    atomicAdd(&s[idx], it);
    idx = (idx + 97) & 16383;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[5];
}
__global__ void k_rmw(int* out, int iters, int stride) {
  extern __shared__ int s[];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) s[i] = 0;
  __syncthreads();
  unsigned idx = (threadIdx.x * stride) & 16383;
  for (int it = 0; it < iters; ++it) {
    s[idx] += it;
    idx = (idx + 97) & 16383;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[5];
}
int main() {
  int* d; cudaMalloc(&d, 4096 * 4);
  cudaFuncSetAttribute(k_atoms, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(k_rmw, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096, threads = 512, blocks = sms * 2;
  for (int stride : {1, 33}) {
    for (int which = 0; which < 2; ++which) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (which == 0) k_atoms<<<blocks, threads, 65536>>>(d, iters, stride);
        else k_rmw<<<blocks, threads, 65536>>>(d, iters, stride);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = (double)blocks * threads * iters;
        if (rep) printf("%s stride %d: %.3f ms, %.2f G lane-ops/s, %.3f lane-ops/clk/SM @1.9GHz\n", which ? "LDS/STS rmw" : "ATOMS.ADD", stride, ms, ops / ms / 1e6, ops / (ms * 1e-3) / sms / 1.9e9);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
