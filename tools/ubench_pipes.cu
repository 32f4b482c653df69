// Pipe-assignment microbenchmark: which SASS ops share the ALU pipe on B200.
// Each kernel runs a long chain of independent ops (8 accumulators, no
// memory); a pair kernel interleaves two ops: time(pair) ~ max(a, b) means
// different pipes, ~ a + b the same pipe.   nvcc -arch=sm_100a -O3 -o x x.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

#define N_IT 4096
#define OP_LOP3(x, y) asm volatile("lop3.b32 %0, %0, %1, 0x1234, 0x96;" : "+r"(x) : "r"(y))
#define OP_PRMT(x, y) asm volatile("prmt.b32 %0, %0, %1, 0x5432;" : "+r"(x) : "r"(y))
#define OP_VMIN(x, y) asm volatile("min.u16x2 %0, %0, %1;" : "+r"(x) : "r"(y))
#define OP_HMIN(x, y) asm volatile("min.f16x2 %0, %0, %1;" : "+r"(x) : "r"(y))
#define OP_HSET(x, y) asm volatile("set.le.f16x2.f16x2 %0, %0, %1;" : "+r"(x) : "r"(y))
#define OP_HADD(x, y) asm volatile("add.f16x2 %0, %0, %1;" : "+r"(x) : "r"(y))
#define OP_HFMA(x, y) asm volatile("fma.rn.f16x2 %0, %0, %1, %1;" : "+r"(x) : "r"(y))
#define OP_IMAD(x, y) asm volatile("mad.lo.u32 %0, %0, %1, %1;" : "+r"(x) : "r"(y))
#define OP_IADD(x, y) asm volatile("add.u32 %0, %0, %1;" : "+r"(x) : "r"(y))
#define OP_IADD3(x, y) asm volatile("{.reg .u32 t; add.u32 t, %0, %1; sub.u32 %0, t, 0x777;}" : "+r"(x) : "r"(y))
#define OP_SHF(x, y) asm volatile("shf.r.wrap.b32 %0, %0, %1, 15;" : "+r"(x) : "r"(y))
#define OP_SHR(x, y) asm volatile("shr.u32 %0, %0, 15;" : "+r"(x))
#define OP_MULHI(x, y) asm volatile("mul.hi.u32 %0, %0, 65536;" : "+r"(x))
#define OP_SEL(x, y) asm volatile("{.reg .pred p; setp.ne.u32 p, %1, 0; selp.b32 %0, %0, %1, p;}" : "+r"(x) : "r"(y))
#define OP_FFMA(x, y) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+r"(x) : "r"(y))
#define OP_FMNMX(x, y) asm volatile("min.f32 %0, %0, %1;" : "+r"(x) : "r"(y))
#define OP_IMNMX(x, y) asm volatile("min.u32 %0, %0, %1;" : "+r"(x) : "r"(y))
#define OP_LEAHI(x, y) asm volatile("{.reg .u32 t; shr.u32 t, %1, 16; add.u32 %0, %0, t;}" : "+r"(x) : "r"(y))
#define OP_F2I(x, y) asm volatile("{.reg .f32 f; mov.b32 f, %0; cvt.rmi.u32.f32 %0, f;}" : "+r"(x))
#define OP_VSUB(x, y) asm volatile("sub.u16x2 %0, %0, %1;" : "+r"(x) : "r"(y))
#define OP_VADD(x, y) asm volatile("add.u16x2 %0, %0, %1;" : "+r"(x) : "r"(y))

#define K1(NAME, OP)                                                                \
    __global__ void k_##NAME(uint32_t* out, uint32_t s) {                          \
        uint32_t a0 = s ^ threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7; \
        _Pragma("unroll 2") for (int i = 0; i < N_IT; ++i) { OP(a0, s); OP(a1, s); OP(a2, s); OP(a3, s); OP(a4, s); OP(a5, s); OP(a6, s); OP(a7, s); } \
        out[blockIdx.x * blockDim.x + threadIdx.x] = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7; }
#define K2(NAME, OPA, OPB)                                                          \
    __global__ void k_##NAME(uint32_t* out, uint32_t s) {                          \
        uint32_t a0 = s ^ threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7; \
        uint32_t b0 = a0 * 3, b1 = b0 + 1, b2 = b0 + 2, b3 = b0 + 3, b4 = b0 + 4, b5 = b0 + 5, b6 = b0 + 6, b7 = b0 + 7; \
        _Pragma("unroll 2") for (int i = 0; i < N_IT; ++i) { OPA(a0, s); OPB(b0, s); OPA(a1, s); OPB(b1, s); OPA(a2, s); OPB(b2, s); OPA(a3, s); OPB(b3, s); \
                                          OPA(a4, s); OPB(b4, s); OPA(a5, s); OPB(b5, s); OPA(a6, s); OPB(b6, s); OPA(a7, s); OPB(b7, s); } \
        out[blockIdx.x * blockDim.x + threadIdx.x] = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7 ^ b0 ^ b1 ^ b2 ^ b3 ^ b4 ^ b5 ^ b6 ^ b7; }

K1(lop3, OP_LOP3) K1(prmt, OP_PRMT) K1(vmin, OP_VMIN) K1(hmin, OP_HMIN) K1(hset, OP_HSET) K1(hadd, OP_HADD)
K1(hfma, OP_HFMA) K1(imad, OP_IMAD) K1(iadd, OP_IADD) K1(iadd3, OP_IADD3) K1(shf, OP_SHF) K1(shr, OP_SHR)
K1(mulhi, OP_MULHI) K1(sel, OP_SEL) K1(ffma, OP_FFMA) K1(fmnmx, OP_FMNMX) K1(imnmx, OP_IMNMX) K1(leahi, OP_LEAHI)
K1(f2i, OP_F2I)
K2(lop3_imad, OP_LOP3, OP_IMAD) K2(lop3_hset, OP_LOP3, OP_HSET) K2(lop3_hadd, OP_LOP3, OP_HADD)
K2(lop3_vmin, OP_LOP3, OP_VMIN) K2(lop3_hmin, OP_LOP3, OP_HMIN) K2(lop3_prmt, OP_LOP3, OP_PRMT)
K2(lop3_iadd, OP_LOP3, OP_IADD) K2(lop3_shf, OP_LOP3, OP_SHF) K2(lop3_ffma, OP_LOP3, OP_FFMA)
K2(lop3_mulhi, OP_LOP3, OP_MULHI) K2(lop3_fmnmx, OP_LOP3, OP_FMNMX) K2(lop3_imnmx, OP_LOP3, OP_IMNMX)
K2(lop3_sel, OP_LOP3, OP_SEL) K2(lop3_f2i, OP_LOP3, OP_F2I) K2(imad_hset, OP_IMAD, OP_HSET)
K2(imad_hadd, OP_IMAD, OP_HADD) K2(ffma_hadd, OP_FFMA, OP_HADD)
K2(lop3_shr, OP_LOP3, OP_SHR)

typedef void (*KF)(uint32_t*, uint32_t);
int main() {
    uint32_t* out;
    cudaMalloc(&out, 148 * 8 * 1024 * 4);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    struct { const char* n; KF f; int ops; } ks[] = {
#define E1(N) {#N, k_##N, 8}
#define E2(N) {#N, k_##N, 16}
        E1(lop3), E1(prmt), E1(vmin), E1(hmin), E1(hset), E1(hadd), E1(hfma), E1(imad), E1(iadd), E1(iadd3), E1(shf),
        E1(shr), E1(mulhi), E1(sel), E1(ffma), E1(fmnmx), E1(imnmx), E1(leahi), E1(f2i),
        E2(lop3_imad), E2(lop3_hset), E2(lop3_hadd), E2(lop3_vmin), E2(lop3_hmin), E2(lop3_prmt), E2(lop3_iadd),
        E2(lop3_shf), E2(lop3_ffma), E2(lop3_mulhi), E2(lop3_fmnmx), E2(lop3_imnmx), E2(lop3_sel), E2(lop3_f2i),
        E2(imad_hset), E2(imad_hadd), E2(ffma_hadd), E2(lop3_shr)};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (auto& k : ks) {
        const int blocks = nsm * 8, threads = 256;  // 64 warps / SM
        k.f<<<blocks, threads>>>(out, 7);
        cudaEventRecord(e0);
        k.f<<<blocks, threads>>>(out, 7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        double warp_ops = (double)blocks * threads / 32 * N_IT * k.ops;
        double per_sm_clk = warp_ops / nsm / (ms * 1e-3 * clk * 1e3);
        printf("%-12s %8.3f ms  %5.2f warp-instr/SM/clk (ops counted: %d per iter)\n", k.n, ms, per_sm_clk, k.ops);
    }
    return 0;
}
