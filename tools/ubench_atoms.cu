// Shared-memory atomic throughput on this GPU (design input for the
// histogram kernels).  Each CTA hammers a 40 x 513 u32 shared histogram with
// one of several address patterns; reports warp-ATOMS per SM per clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

template <int PATTERN, int WIDE>
__global__ void kern(int iters, unsigned long long* out, long long* cycles) {
  extern __shared__ uint32_t h[];
  const int N = 40 * 513;
  for (int i = threadIdx.x; i < N * (WIDE ? 2 : 1); i += blockDim.x) h[i] = 0;
  __syncthreads();
  long long t0 = clock64();
  uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t s = hash32(threadIdx.x * 7919 + blockIdx.x);
  for (int it = 0; it < iters; ++it) {
    uint32_t a;
    if (PATTERN == 0) a = (warp * 32 + lane + it * 97) % N;                 // distinct banks
    else if (PATTERN == 1) { s = hash32(s + it); a = s % N; }               // random
    else if (PATTERN == 2) a = (it * 131 + warp) % N;                        // same address per warp
    else { s = hash32(s + it); a = (s % 24) * 513 + ((it * 7 + lane / 3) % 400); } // smooth-like: ~11 distinct per warp
    if (WIDE) atomicAdd(reinterpret_cast<unsigned long long*>(h) + a, 1ull);
    else atomicAdd(&h[a], 1u);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) { cycles[blockIdx.x] = t1 - t0; }
  if (threadIdx.x == 0) atomicAdd(out, (unsigned long long)h[0]);
}

template <int P, int W>
void run(const char* name, int blocks_per_sm, int threads) {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int grid = nsm * blocks_per_sm, iters = 4096;
  size_t smem = 40 * 513 * 4 * (W ? 2 : 1);
  cudaFuncSetAttribute(kern<P, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned long long* out; long long* cyc; cudaMalloc(&out, 8); cudaMalloc(&cyc, 8 * grid);
  kern<P, W><<<grid, threads, smem>>>(iters, out, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<P, W><<<grid, threads, smem>>>(iters, out, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double warp_atoms_per_sm = (double)blocks_per_sm * threads / 32 * iters;
  printf("%-28s blk/SM=%d thr=%d: %.3f ms, %.2f warp-ATOMS/SM/clk (clk of blk0), %.1f G lane-atomics/s\n", name,
         blocks_per_sm, threads, ms, warp_atoms_per_sm / c, (double)grid * threads * iters / ms / 1e6);
  cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
}

int main() {
  run<0, 0>("u32 distinct banks", 2, 512);
  run<1, 0>("u32 random", 2, 512);
  run<2, 0>("u32 same addr per warp", 2, 512);
  run<3, 0>("u32 smooth-like (~11/warp)", 2, 512);
  run<0, 1>("u64 distinct", 1, 512);
  run<1, 1>("u64 random", 1, 512);
  return 0;
}
