// ft_lattice.cuh -- helpers shared by the fused-curve kernels (ft_lattice.cu,
// ft_lines.cu): packed 16-bit level pairs, fused quantize of a k-adjacent
// cell pair, launch geometry and work planning.  sm_100a only.
#pragma once
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "ft_common.cuh"

namespace ft {

constexpr int LTW = 32;              // staged words per tile row (one warp)
constexpr int LTJ = 16;              // staged rows (warps)
constexpr int LNT = LTW * LTJ;       // 512 threads, one staged word each
constexpr int LCW = LTW - 1;         // compute words per row (31 -> 62 lattice columns)
constexpr int LCJ = LTJ - 1;         // compute rows (15)


struct LGeo {
    int64_t H, W, D, v0, v1, first, bstride;
    int M, tiles_j, tiles_k, chunk, hs;
    int64_t n_items, items_per_image;
    int ti_j0, ti_j1, ti_k0, ti_k1;  // ft_lines3d: interior tile ranges (guard-free kernel)
    int hk;                          // ft_lines3d: signature row stride / 255
    int rf_n, rf_j0[4];              // ft_lines3d: the row-boundary warp strips (j0 values)
    int kb_lo, kb_hi;                // ft_lines3d: k-boundary column tiles at each end
    int e_chunk;                     // ft_lines3d: planes per boundary warp item
    int64_t e_items;                 // ft_lines3d: boundary warp items
    uint32_t four;                   // line kernels: 4 as an opaque register (the quantizer's IMAD, not LEA)
};

__device__ __forceinline__ uint32_t vmin2(uint32_t a, uint32_t b) { return __vminu2(a, b); }
__device__ __forceinline__ uint32_t vmax2(uint32_t a, uint32_t b) { return __vmaxu2(a, b); }
// (hi half of a, lo half of b): the pair shifted down by one cell
__device__ __forceinline__ uint32_t shift_pair(uint32_t a, uint32_t b) { return __byte_perm(a, b, 0x5432); }

// w holds two byte offsets (level * 4 * CP + copy * 4) of two lattice points;
// row bases are uniform, so each event is one extract + one ATOMS
__device__ __forceinline__ void inc2(char* __restrict__ h, int row, int hs, uint32_t w)
{
    char* base = h + row * hs;
    ft_check_smem((uint32_t)__cvta_generic_to_shared(base + (w & 0xFFFFu)));
    ft_check_smem((uint32_t)__cvta_generic_to_shared(base + (w >> 16)));
    atomicAdd(reinterpret_cast<uint32_t*>(base + (w & 0xFFFFu)), 1u);
    atomicAdd(reinterpret_cast<uint32_t*>(base + (w >> 16)), 1u);
}

// Histograms are privatised CP ways by lane: bin (level, copy) sits at
// (level * CP + copy) words, copy = lane % CP, so two lanes can only meet in
// a bank if they share lane % CP -- the bank-conflict degree of the event
// ATOMS drops from ~2.2 wavefronts to ~1 (profiles/r01).  The copy offset is
// added to the loaded level words once per step (mins commute with it).
template <int CP>
struct Priv {
    static constexpr int SH = CP == 8 ? 3 : CP == 4 ? 2 : CP == 2 ? 1 : 0;
};

template <int DT>
struct Pair;
template <> struct Pair<FT_F32> { using T = float2; };
template <> struct Pair<FT_I32> { using T = int2; };
template <> struct Pair<FT_U16> { using T = ushort2; };
template <> struct Pair<FT_U8> { using T = uchar2; };

// Two k-adjacent cells (k, k+1), k even.  VEC (even extent): both cells share
// validity and one aligned 2-element load fetches them; otherwise each cell
// is checked and loaded on its own.
template <int DT, bool VEC>
__device__ __forceinline__ typename Pair<DT>::T load_pair(const typename Elem<DT>::T* p, bool okx, bool oky)
{
    typename Pair<DT>::T v{};
    if constexpr (VEC) {
        if (okx) v = __ldg(reinterpret_cast<const typename Pair<DT>::T*>(p));
    } else {
        if (okx) v.x = __ldg(p);
        if (oky) v.y = __ldg(p + 1);
    }
    return v;
}

// Branch-free: quantize both cells unconditionally, then select the sentinel.
// Output lanes hold level * 4 << SH (byte offsets of copy 0).
template <int DT, int QM, int SH>
__device__ __forceinline__ uint32_t pack_pair(const typename Pair<DT>::T& v, bool okx, bool oky, const float* tt,
                                              const QuantDev& q, int M, uint32_t sent)
{
    uint32_t a = to_level4<DT, QM>(v.x, tt, q.scale, q.bias, q.negate, M) << SH;
    uint32_t b = to_level4<DT, QM>(v.y, tt, q.scale, q.bias, q.negate, M) << SH;
    a = okx ? a : sent;
    b = oky ? b : sent;
    return __byte_perm(a, b, 0x5410);
}

// float -> u16 with floor, saturating (PTX float-to-int conversions saturate).
__device__ __forceinline__ uint32_t f2u16_rd(float f)
{
    unsigned short r;
    asm("cvt.rmi.u16.f32 %0, %1;" : "=h"(r) : "f"(f));
    return r;
}

// Packed-pair quantization for FT_Q_POW2: both cells converted with a
// saturating floor to u16, then clamped to M, scaled to byte offsets and
// masked to the sentinel as one 32-bit word (keep = 0xFFFF per present cell).
template <int DT>
__device__ __forceinline__ uint32_t pack_pair_pow2(const typename Pair<DT>::T& v, uint32_t keep, float scale,
                                                   uint32_t Mpk, uint32_t sent2)
{
    const uint32_t a = f2u16_rd(__fmaf_rd((float)v.x, scale, 0.5f));
    const uint32_t b = f2u16_rd(__fmaf_rd((float)v.y, scale, 0.5f));
    const uint32_t w = __vminu2(__byte_perm(a, b, 0x5410), Mpk) << 2;
    return (w & keep) | (sent2 & ~keep);
}

// Sum the CP copies of every (row, level) bin into the global histogram.
template <int CP>
__device__ __forceinline__ void flush_rows(uint32_t* h, unsigned long long* __restrict__ out, int nrows, int M2,
                                           int hs_words, bool zero)
{
    for (int i = threadIdx.x; i < nrows * M2; i += blockDim.x) {
        const int r = i / M2, l = i - r * M2;
        uint32_t* p = h + r * hs_words + l * CP;
        uint32_t v = 0;
#pragma unroll
        for (int c = 0; c < CP; ++c) {
            v += p[c];
            if (zero) p[c] = 0;
        }
        if (v) atomicAdd(&out[i], (unsigned long long)v);
    }
}

static int nsm_l()
{
    int dev = 0, n = kSMs;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

static QuantDev qdev(const ft_quant* qa)
{
    return QuantDev{qa ? qa->mode : FT_Q_IDENTITY, qa ? qa->negate : 0, qa ? qa->scale : 0.f, qa ? qa->bias : 0.f,
                    qa ? qa->thresholds : nullptr, 0.f};
}

// histogram row stride in bytes for cp copies (16-byte aligned rows)
static int row_stride(int M, int cp) { return ((M + 2) * 4 * cp + 15) / 16 * 16; }

// Work split: tiles x row-chunks, contiguous item ranges per CTA, enough
// items (>= ~6 per CTA) to balance while keeping marches long.
static void plan_items(LGeo& g, int64_t tiles, int64_t batch, int64_t grid_cap, int64_t min_rows)
{
    const int64_t rows = g.v1 - g.v0;
    int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>(cdiv(6 * grid_cap, tiles * batch), rows / min_rows));
    g.chunk = (int)cdiv(rows, nchunks);
    nchunks = cdiv(rows, g.chunk);
    g.items_per_image = tiles * nchunks;
    g.n_items = g.items_per_image * batch;
}

// halo: low planes needed below v0 (1 for the 2D kernels, 2 for 3D: the
// signature kernel reads the -i neighbour of plane v0-1)
static bool window_ok(const ft_window* win, int64_t H, int64_t v0, int64_t v1, int halo = 1)
{
    const int64_t need_lo = std::max<int64_t>(v0 - halo, 0), need_hi = std::min<int64_t>(v1 - 1, H - 1);
    return !(need_lo <= need_hi &&
             (win->data == nullptr || need_lo < win->first || need_hi >= win->first + win->count));
}

}  // namespace ft
