// Shared-memory atomic throughput on this GPU (design input for the
// histogram kernels).  Addresses are precomputed into registers so the loop
// is ATOMS-only; reports warp-ATOMS per SM per clock for several patterns.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

constexpr int NA = 16;  // addresses per thread

template <int PATTERN, int INC>
__global__ void kern(int iters, unsigned long long* out, long long* cycles, int nbins) {
  extern __shared__ uint32_t h[];
  for (int i = threadIdx.x; i < nbins; i += blockDim.x) h[i] = 0;
  uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t a[NA];
#pragma unroll
  for (int q = 0; q < NA; ++q) {
    uint32_t r = hash32(threadIdx.x * 131 + q * 7919 + blockIdx.x * 3);
    uint32_t v;
    if (PATTERN == 0) v = (q * 32 + lane) % nbins;                       // distinct banks, distinct addr
    else if (PATTERN == 1) v = r % nbins;                                // random
    else if (PATTERN == 2) v = (q * 37 + warp * 5) % nbins;              // one address per warp
    else if (PATTERN == 3) v = ((q * 97 + warp * 13) % (nbins - 64)) + lane / 2 + (r & 7);  // smooth: ~20 distinct, clustered
    else v = (q * 64 + lane * 2) % nbins;                                // 2-way bank conflict
    a[q] = v;
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      if (INC) atomicAdd(&h[a[q]], 1u);
      else atomicAdd(&h[a[q]], lane + 1u);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (threadIdx.x == 0) atomicAdd(out, (unsigned long long)h[0]);
}

template <int P, int I>
void run(const char* name, int bps, int threads, int nbins) {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int grid = nsm * bps, iters = 256;
  size_t smem = nbins * 4;
  cudaFuncSetAttribute(kern<P, I>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long* out; long long* cyc; cudaMalloc(&out, 8); cudaMalloc(&cyc, 8 * grid);
  kern<P, I><<<grid, threads, smem>>>(iters, out, cyc, nbins);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<P, I><<<grid, threads, smem>>>(iters, out, cyc, nbins);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double wa = (double)bps * threads / 32 * iters * NA;
  printf("%-34s bins=%6d: %.3f ms, %.3f warp-ATOMS/SM/clk, %.0f G lane-atomics/s\n", name, nbins, ms, wa / c,
         (double)grid * threads * iters * NA / ms / 1e6);
  cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
}

int main() {
  for (int bins : {1536, 20520}) {
    run<0, 1>("inc distinct banks", 2, 512, bins);
    run<4, 1>("inc 2-way bank conflict", 2, 512, bins);
    run<1, 1>("inc random", 2, 512, bins);
    run<3, 1>("inc smooth-clustered", 2, 512, bins);
    run<2, 1>("inc same address per warp", 2, 512, bins);
    run<0, 0>("add(reg) distinct banks", 2, 512, bins);
    run<1, 0>("add(reg) random", 2, 512, bins);
    run<3, 0>("add(reg) smooth-clustered", 2, 512, bins);
    run<2, 0>("add(reg) same address per warp", 2, 512, bins);
  }
  return 0;
}
