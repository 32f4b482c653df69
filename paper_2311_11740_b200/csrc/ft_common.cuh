// ft_common.cuh -- shared device helpers for the fieldtopo-b200 kernels.
//
// Level decoding (fused quantize), sorting networks and launch bookkeeping.
// Everything here is sm_100a device code; see DESIGN.md §3 for the layout.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fieldtopo_b200.h"

#define FT_CUDA_TRY(expr)                                   \
    do {                                                    \
        cudaError_t _e = (expr);                            \
        if (_e != cudaSuccess) return FT_ERR_CUDA_BASE + (int)_e; \
    } while (0)

namespace ft {

constexpr int kSMs = 148;

// ------------------------------------------------ opt-in shared-memory checks
// compute-sanitizer is unavailable on the GPU pool, so a build with
// -DFT_BOUNDS_CHECK (tools/dev/build_checked.py) traps on any shared-memory
// histogram update outside its block: ft_sh_add checks a row index against
// the histogram's extent, ft_check_smem an absolute shared-window address
// (the line kernels' packed 16-bit addresses) against the dynamic block.
// The product build compiles both to the bare atomic.
#ifdef FT_BOUNDS_CHECK
__device__ __forceinline__ void ft_check_smem(uint32_t addr)
{
    extern __shared__ unsigned char ft_dyn_smem_chk[];
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(ft_dyn_smem_chk);
    uint32_t size;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(size));
    if (addr < base || addr + 4u > base + size || (addr & 3u)) __trap();
}
__device__ __forceinline__ void ft_sh_add(uint32_t* h, uint32_t i, uint32_t n)
{
    if (i >= n) __trap();
    atomicAdd(&h[i], 1u);
}
#else
__device__ __forceinline__ void ft_check_smem(uint32_t) {}
__device__ __forceinline__ void ft_sh_add(uint32_t* h, uint32_t i, uint32_t) { atomicAdd(&h[i], 1u); }
#endif
// increment / load at an absolute shared-window address (the map kernels'
// keys carry the histogram's shared address, so a bin address is a mask or a
// shift of the sorted key)
__device__ __forceinline__ void ft_sh_inc(uint32_t addr)
{
    ft_check_smem(addr);
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
}
__device__ __forceinline__ uint32_t ft_sh_ld(uint32_t addr)
{
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// ------------------------------------------------------------------ loads
template <int DT> struct Elem;
template <> struct Elem<FT_I32> { using T = int32_t; };
template <> struct Elem<FT_U8> { using T = uint8_t; };
template <> struct Elem<FT_U16> { using T = uint16_t; };
template <> struct Elem<FT_F32> { using T = float; };
template <> struct Elem<FT_F64> { using T = double; };

// Streaming read-only load: the field is read once per kernel (halo re-reads
// hit L2), so keep it out of L1.
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) { return __ldg(p); }

// ------------------------------------------------------------ quantization
// Quantization state for one launch.  The float64 reference formula
// (fields.py:20-33) is monotone, so a host-built float32 threshold table
// tt[0..M+1] (tt[0] = -inf, tt[l] = smallest x with level(x) >= l,
// tt[M+1] = NaN) decides it exactly: level(x) = #{l >= 1 : x >= tt[l]}.
// FT_Q_TABLE: the host guarantees the float32 estimate
// est = clamp(floor(fmaf(x, scale, bias)), 0, M) is the level L or L - 1
// (bias = -lo * scale, estimate error < 0.5 level), so ONE comparison fixes it.
// FT_Q_TABLE_ROBUST (ill-conditioned ranges) walks the table both ways.
struct QuantDev {
    int mode;        // FT_Q_IDENTITY / FT_Q_TABLE / FT_Q_TABLE_ROBUST
    int negate;      // reversed range (hi < lo): evaluate on -x
    float scale, bias;
    const float* tt; // device, M+2 entries (kernels stage a shared copy)
    float inv;       // FT_Q_POW2: 1 / hi (exact, a power of two), set per launch
    // FT_Q_UMAGIC (internal: uint8 / uint16 inputs, integer range lo < hi):
    // level = ((clamp(x, lo, hi) - lo) * u_mul + u_add) * u_magic >> (32 + u_shift)
    uint32_t u_lo2, u_hi2;  // lo, hi in both 16-bit halves
    uint32_t u_mul, u_add, u_magic, u_shift;
};
constexpr int FT_Q_UMAGIC = 4;  // internal quantizer mode, never in an ft_quant

template <int DT, int QM>
__device__ __forceinline__ uint32_t to_level(typename Elem<DT>::T raw, const float* __restrict__ tt,
                                             float scale, float bias, int negate, int M)
{
    if constexpr (QM == FT_Q_IDENTITY) {
        // Identity levels are validated on the host (Field2D/Field3D); clamp
        // to the sentinel so a bad level can never index past the histogram.
        uint32_t v = (uint32_t)raw;
        return min(v, (uint32_t)(M + 1));
    } else {
        float x = (float)raw;
        if constexpr (QM == FT_Q_TABLE_ROBUST) {
            if (negate) x = -x;  // FT_Q_TABLE is never used for reversed ranges
        }
        int est = __float2int_rd(fmaf(x, scale, bias));
        est = min(max(est, 0), M);
        if constexpr (QM == FT_Q_TABLE) {
            est += (x >= tt[est + 1]) ? 1 : 0;
        } else {
            while (est < M && x >= tt[est + 1]) ++est;
            while (est > 0 && x < tt[est]) --est;
        }
        return (uint32_t)est;
    }
}

// level * 4 (a shared-memory byte offset), for the 16-bit packed kernels.
// FT_Q_POW2 (lo = 0, hi = 2^p, scale = M / hi exact): the reference's float64
// (x - 0) * M / hi + 0.5 is exact for every float32 x (<= 47 significant
// bits), so level = clamp(floor(x * scale + 0.5)).  The FMA rounded toward
// -infinity never crosses an integer upward and every integer below 2^24 is a
// float, so floor(fma_rd(x, scale, 0.5)) IS that floor: three instructions,
// no table, no shared-memory load.
template <int DT, int QM>
__device__ __forceinline__ uint32_t to_level4(typename Elem<DT>::T raw, const float* __restrict__ tt, float scale,
                                              float bias, int negate, int M)
{
    if constexpr (QM == FT_Q_POW2) {
        const float x = (float)raw;
        const uint32_t est = __float2uint_rd(__fmaf_rd(x, scale, 0.5f));  // saturates < 0 and NaN to 0
        return min(est, (uint32_t)M) << 2;
    } else if constexpr (QM == FT_Q_TABLE) {
        const float x = (float)raw;
        // unsigned floor conversion saturates negatives (and NaN) to 0: one clamp
        const uint32_t est = min(__float2uint_rd(fmaf(x, scale, bias)), (uint32_t)M);
        const uint32_t e4 = est << 2;
        const float t = *reinterpret_cast<const float*>(reinterpret_cast<const char*>(tt) + e4 + 4);
        return x >= t ? e4 + 4 : e4;
    } else {
        return to_level<DT, QM>(raw, tt, scale, bias, negate, M) << 2;
    }
}

// float64 inputs (ft_quantize only): the same scheme with a double table.
template <int QM>
__device__ __forceinline__ uint32_t to_level_f64(double x, const double* __restrict__ tt, double scale,
                                                 double bias, int negate, int M)
{
    if (negate) x = -x;
    double y = fma(x, scale, bias);
    int est = (y != y) ? 0 : (y <= 0.0 ? 0 : (y >= (double)M ? M : (int)floor(y)));
    if constexpr (QM == FT_Q_TABLE) {
        est += (x >= tt[est + 1]) ? 1 : 0;
    } else {
        while (est < M && x >= tt[est + 1]) ++est;
        while (est > 0 && x < tt[est]) --est;
    }
    return (uint32_t)est;
}

// ------------------------------------------------------- sorting networks
__device__ __forceinline__ void cswap(uint32_t& a, uint32_t& b)
{
    uint32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}

// Optimal 5-comparator network for 4 keys.
__device__ __forceinline__ void sort4(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d)
{
    cswap(a, b);
    cswap(c, d);
    cswap(a, c);
    cswap(b, d);
    cswap(b, c);
}

// Batcher odd-even merge of two sorted 4-sequences (9 comparators).
__device__ __forceinline__ void merge44(uint32_t* k)
{
    // k[0..3] sorted, k[4..7] sorted
    cswap(k[0], k[4]);
    cswap(k[1], k[5]);
    cswap(k[2], k[6]);
    cswap(k[3], k[7]);
    cswap(k[2], k[4]);
    cswap(k[3], k[5]);
    cswap(k[1], k[2]);
    cswap(k[3], k[4]);
    cswap(k[5], k[6]);
}

// Odd-even merge of two sorted pairs (3 comparators).
__device__ __forceinline__ void merge22(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d)
{
    cswap(a, c);
    cswap(b, d);
    cswap(b, c);
}

// FT_Q_TABLE assumes an increasing range; reversed ranges take the walking path.
inline int effective_qmode(const ft_quant* q, bool pow2_ok = false)
{
    if (!q) return FT_Q_IDENTITY;
    if (q->mode == FT_Q_POW2) return (pow2_ok && !q->negate) ? FT_Q_POW2 : FT_Q_TABLE;
    return (q->mode == FT_Q_TABLE && q->negate) ? FT_Q_TABLE_ROBUST : q->mode;
}

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace ft
