// ubench_tiles.cu -- load-pattern microbenchmark for the 2D line kernel
// (ft_lines2d.cu): how many DRAM bytes and how much time does a streaming
// read of a C2-sized f32 image (8192 x 8192) cost with
//   mis : the shipping tiling -- 62-column tiles, each warp row reads the
//         64-cell window starting at column 62 t - 2 (misaligned to 64 B)
//   al  : 64-column tiles read as aligned 256-byte segments
//   alh : al plus the two halo pairs (64 t - 2 .. 64 t - 1, 64 t + 64 ..
//         64 t + 65) loaded by lanes 0 and 31 every row
// Same work split as lines2d_kernel (pieces of 96 rows x one tile, even cut
// over 148 CTAs x 16 warps, 8 rows in flight per lane).  Cold L2 per rep
// (a 512 MiB buffer is rewritten between reps).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/ubench_tiles tools/ubench_tiles.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int H = 8192, W = 8192, RB = 96, PF = 8, NTH = 512;

// IL: pieces of a CTA's range dealt round-robin to its 16 warps (warp w takes
// pieces w, w + 16, ...), so the warps march adjacent tiles of the same rows
// at about the same time; otherwise each warp takes a contiguous sub-range.
template <int MODE, bool IL>
__global__ void __launch_bounds__(NTH, 1) stream_tiles(const float* __restrict__ img, float* __restrict__ out)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int TW = MODE == 0 ? 62 : 64;
    const int ntiles = MODE == 0 ? (W + 1) / 62 + 1 : W / 64;
    const int64_t npieces = (int64_t)((H + RB - 1) / RB) * ntiles;
    const int64_t P0 = npieces * blockIdx.x / gridDim.x, P1 = npieces * (blockIdx.x + 1) / gridDim.x;
    const int64_t wa = IL ? P0 + warp : P0 + (P1 - P0) * warp / 16;
    const int64_t we = IL ? P1 : P0 + (P1 - P0) * (warp + 1) / 16;
    float acc = 0.f;
    for (int64_t piece = wa; piece < we; piece += IL ? 16 : 1) {
        const int64_t rb = piece / ntiles;
        const int t = (int)(piece - rb * ntiles);
        const int r0 = (int)(rb * RB), r1 = (int)min((int64_t)r0 + RB, (int64_t)H);
        int kc = MODE == 0 ? t * TW - 2 + 2 * lane : t * TW + 2 * lane;
        kc = min(max(kc, 0), W - 2);
        int kh = lane == 0 ? t * 64 - 2 : t * 64 + 64;
        kh = min(max(kh, 0), W - 2);
        const float* p = img + (int64_t)r0 * W + kc;
        const float* ph = img + (int64_t)r0 * W + kh;
        float2 buf[PF], hb[PF];
#pragma unroll
        for (int i = 0; i < PF; ++i) {
            if (r0 + i < r1) buf[i] = *reinterpret_cast<const float2*>(p + (int64_t)i * W);
            if (MODE == 2 && (lane == 0 || lane == 31) && r0 + i < r1)
                hb[i] = *reinterpret_cast<const float2*>(ph + (int64_t)i * W);
        }
        int s = r0;
        for (; s + 2 * PF <= r1; s += PF) {  // steady state: no guards
#pragma unroll
            for (int i = 0; i < PF; ++i) {
                acc += buf[i].x * 1.0001f + buf[i].y;
                if (MODE == 2 && (lane == 0 || lane == 31)) acc += hb[i].x - hb[i].y;
                buf[i] = *reinterpret_cast<const float2*>(p + (int64_t)(s + i + PF - r0) * W);
                if (MODE == 2 && (lane == 0 || lane == 31))
                    hb[i] = *reinterpret_cast<const float2*>(ph + (int64_t)(s + i + PF - r0) * W);
            }
        }
        for (; s < r1; s += PF) {
#pragma unroll
            for (int i = 0; i < PF; ++i) {
                if (s + i < r1) {
                    acc += buf[i].x * 1.0001f + buf[i].y;
                    if (MODE == 2 && (lane == 0 || lane == 31)) acc += hb[i].x - hb[i].y;
                    const int nr = s + i + PF;
                    if (nr < r1) {
                        buf[i] = *reinterpret_cast<const float2*>(p + (int64_t)(nr - r0) * W);
                        if (MODE == 2 && (lane == 0 || lane == 31))
                            hb[i] = *reinterpret_cast<const float2*>(ph + (int64_t)(nr - r0) * W);
                    }
                }
            }
        }
    }
    out[blockIdx.x * NTH + threadIdx.x] = acc;
}

__global__ void flush(float* b, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] += 1.f;
}

int main()
{
    float *img, *out, *fl;
    const size_t n = (size_t)H * W, nf = (512u << 20) / 4;
    cudaMalloc(&img, n * 4);
    cudaMalloc(&out, 148 * NTH * 4);
    cudaMalloc(&fl, nf * 4);
    cudaMemset(img, 0, n * 4);
    cudaMemset(fl, 0, nf * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[6] = {"mis (62-col tiles, 64-cell window at 62t-2)", "al (64-col aligned)",
                            "alh (aligned + halo pairs, lanes 0/31)", "mis-il (warps interleaved over pieces)",
                            "al-il", "alh-il"};
    for (int mode = 0; mode < 6; ++mode) {
        float best = 1e9f, sum = 0.f;
        const int reps = 12;
        for (int r = 0; r < reps; ++r) {
            flush<<<592, 512>>>(fl, nf);
            cudaEventRecord(a);
            if (mode == 0) stream_tiles<0, false><<<148, NTH>>>(img, out);
            if (mode == 1) stream_tiles<1, false><<<148, NTH>>>(img, out);
            if (mode == 2) stream_tiles<2, false><<<148, NTH>>>(img, out);
            if (mode == 3) stream_tiles<0, true><<<148, NTH>>>(img, out);
            if (mode == 4) stream_tiles<1, true><<<148, NTH>>>(img, out);
            if (mode == 5) stream_tiles<2, true><<<148, NTH>>>(img, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 2) { best = ms < best ? ms : best; sum += ms; }
        }
        printf("%-48s best %.2f us  mean %.2f us  %.0f GB/s (algorithmic, best)\n", names[mode], best * 1e3,
               sum / (12 - 2) * 1e3, n * 4.0 / (best * 1e-3) / 1e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
