// ft_hist2d.cu -- 2D vertex-contribution transition histograms (map path).
//
// Replaces the reference's _scan_rows_2d (contrib2d.py:161-232).  Vertex
// (i, j) reads cells NW (i-1, j-1), NE (i-1, j), SW (i, j-1), SE (i, j) as
// slots 0..3 (contrib2d.py:39-40); keys level*4 + slot sorted ascending give
// the reference's p0 / p1 / remaining-pair order exactly.  Four events per
// vertex go to 6 transition classes:
//   0: (empty -> q1) @ v0
//   1 / 2: (q1 -> q2 / qd) @ v1      (qd iff p0 + p1 == 3, contrib2d.py:224)
//   3 / 4: (q2 / qd -> q3) @ v2
//   5: (q3 -> q4) @ v3
// hist2d_march (default): a warp marches 62 vertex columns down the rows on
// packed 16-bit keys (two vertices per word) into a per-CTA shared-memory
// histogram, M <= ~7260.  hist2d_wide: any M, one vertex per thread, global
// u64 histogram.  Batches of equally-shaped images (config 3) run in one
// launch with one histogram per image.
#include <algorithm>

#include "ft_common.cuh"
#include "ft_lines.cuh"
#include "ft_tables.h"

namespace ft {

struct Geo2 {
    int64_t H, W, v0, v1, first, batch, bstride;
    int M;
    int tiles;
};

template <int DT, int QM>
__device__ __forceinline__ uint32_t level2(const typename Elem<DT>::T* __restrict__ img, const Geo2& g,
                                           int64_t r, int64_t c, const float* tt, const QuantDev& q)
{
    if (r < 0 || r >= g.H || c < 0 || c >= g.W) return (uint32_t)g.M + 1;
    return to_level<DT, QM>(ld_stream(img + (r - g.first) * g.W + c), tt, q.scale, q.bias, q.negate, g.M);
}

// Any level count (and the fallback when the march's shared histogram does
// not fit): one vertex per thread over every image, row and vertex column,
// keys level*4 + slot in 32 bits, the 4 events booked straight into the
// global u64 histogram of the image.  Thresholds are read from global memory.
template <int DT, int QM>
__global__ void __launch_bounds__(256) hist2d_wide(const typename Elem<DT>::T* __restrict__ buf, Geo2 g,
                                                   QuantDev q, unsigned long long* __restrict__ hist)
{
    const int64_t M2 = g.M + 2;
    const int64_t nj = g.W + 1, rows = g.v1 - g.v0;
    const int64_t n = g.batch * rows * nj;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t % nj;
        const int64_t r = t / nj;
        const int64_t b = r / rows;
        const int64_t i = g.v0 + r % rows;
        const auto* img = buf + b * g.bstride;
        // slots [NW, NE, SW, SE] = 2 di + dj (contrib2d.py:39-40)
        uint32_t k0 = level2<DT, QM>(img, g, i - 1, j - 1, q.tt, q) * 4 + 0;
        uint32_t k1 = level2<DT, QM>(img, g, i - 1, j, q.tt, q) * 4 + 1;
        uint32_t k2 = level2<DT, QM>(img, g, i, j - 1, q.tt, q) * 4 + 2;
        uint32_t k3 = level2<DT, QM>(img, g, i, j, q.tt, q) * 4 + 3;
        sort4(k0, k1, k2, k3);
        unsigned long long* hb = hist + b * (int64_t)FT_NCLASS_2D * M2;
        const bool diag = ((k0 ^ k1) & 3) == 3;  // p0 + p1 == 3 (contrib2d.py:224)
        atomicAdd(&hb[k0 >> 2], 1ull);
        atomicAdd(&hb[(diag ? 2 : 1) * M2 + (k1 >> 2)], 1ull);
        atomicAdd(&hb[(diag ? 4 : 3) * M2 + (k2 >> 2)], 1ull);
        atomicAdd(&hb[5 * M2 + (k3 >> 2)], 1ull);
    }
}

// ------------------------------------------------ register-march map kernel
// The register march of the line kernels: a warp marches a strip of 62 vertex columns down the
// rows, lane l holding the cells (kk, kk+1), kk = k0-1+2l, as packed 16-bit
// level*4 words -- so the keys (level*4 + slot) of the lane's two vertices
// ride in the halves of one word and sort4 / merge22 run once per pair
// (VIMNMX.U16x2).  No staging, no barrier per row; every vertex column
// 0..W is covered (no edge kernel).  Halves outside the vertex range or on a
// halo lane book into a dummy row that is never flushed.
constexpr int HM_NTH = 512;
constexpr int HM_RB = 64;
constexpr int HM_PF = 4;  // rows in flight per lane (even)

__device__ __forceinline__ void hm_cswap2(uint32_t& a, uint32_t& b)
{
    const uint32_t lo = __vminu2(a, b);
    b = __vmaxu2(a, b);
    a = lo;
}

// BA (6 rows of byte offsets fit 16 bits: M <= ~2330): keys are level * 4 +
// slot + 4 per half, so a key with its slot bits masked IS the offset
// rel = (level + 1) * 4 of the level's bin BELOW the top of row 0; the
// histogram grows downward from its top (row r another r * 4 (M + 2) lower,
// the dummy word AT the top), and one IDP.2A per half (sinc2, ft_lines.cuh)
// does the half split, the halo / range select and the address -- no shift,
// no select, no index -> address arithmetic.  Otherwise 16-bit word indices.
template <int DT, int QM, bool VEC, bool EDGE, bool BA>
__device__ __forceinline__ void hm_item(const typename Elem<DT>::T* __restrict__ img, const Geo2& g,
                                        const QuantDev& q, const float* __restrict__ tt, uint32_t* __restrict__ h,
                                        uint32_t hb, int64_t ia, int64_t ib, int k0, int lane)
{
    using P2 = typename Pair<DT>::T;
    using T = typename Elem<DT>::T;
    constexpr uint32_t FULL = 0xFFFFFFFFu, K1 = 0x10001u;
    const int Wi = (int)g.W;
    const uint32_t M2 = (uint32_t)g.M + 2u;
    const uint32_t sent4 = ((uint32_t)g.M + 1u) * 4u;
    const uint32_t hbK = BA ? LINES_REL0 : 0u;  // BA keys: level * 4 + slot + 4
    const uint32_t S = sent4 * K1 + hbK;
    const int kk = k0 - 1 + 2 * lane;
    // vertex columns kk (low half) and kk+1 (high half) that this lane books
    const bool vlo = lane != 0 && kk >= 0 && kk <= Wi, vhi = lane != 31 && kk + 1 >= 0 && kk + 1 <= Wi;
    const uint32_t vmask = __shfl_sync(FULL, (vlo ? 0x0000FFFFu : 0u) | (vhi ? 0xFFFF0000u : 0u), lane);
    const uint32_t vsel = __shfl_sync(FULL, (vlo ? 0x000000FFu : 0u) | (vhi ? 0xFF000000u : 0u), lane);  // sinc2 selector
    const uint32_t top = __shfl_sync(FULL, hb + 24u * M2, lane);  // BA: the top of row 0 = the dummy word
    const uint32_t dummy = 6u * M2 * K1;
    const bool okx = kk >= 0 && kk < Wi, oky = kk + 1 >= 0 && kk + 1 < Wi;
    const int kc = !EDGE ? kk : VEC ? min(max(kk, 0), Wi - 2) : min(max(kk, 0), Wi - 1);
    const int n = (int)(ib - ia);
    // rows t = 0 .. n (row ia-1+t) exist iff t_lo <= t < t_hi; t < tf fetched
    const int t_lo = (int)max((int64_t)0, 1 - ia);
    const int t_hi = (int)min((int64_t)(n + 1), g.H - ia + 1);
    const int tf = t_hi;
    const T* ptr = img + ((ia - 1 - g.first) * g.W + kc);  // row ia-1 (t = 0)

    auto fetch = [&](int t, const T* at, P2& dst) {
        if (t >= t_lo && t < tf) dst = load_pair<DT, VEC>(at, true, EDGE ? kk + 1 < Wi : true);
    };
    auto quant_in = [&](const P2& src) -> uint32_t {
        if constexpr (!EDGE && QM == FT_Q_IDENTITY && (DT == FT_U8 || DT == FT_U16))
            return pack_pair_ident<DT>(src, (sent4 >> 2) * K1, 4u, hbK);  // packed clamp + one multiply-add
        else
            return pack_pair<DT, QM, 0>(src, !EDGE || okx, !EDGE || oky, tt, q, g.M, sent4) + hbK;
    };
    // one vertex row: sorted NW / NE keys of the row above in a, c
    uint32_t a, c;
    auto step = [&](uint32_t V) {
        const uint32_t Wm = shift_pair(__shfl_up_sync(FULL, V, 1), V);
        uint32_t u0 = Wm + 2u * K1, u1 = V + 3u * K1;  // SW, SE
        hm_cswap2(u0, u1);
        uint32_t s0 = a, s1 = c, s2 = u0, s3 = u1;
        hm_cswap2(s0, s2);
        hm_cswap2(s1, s3);
        hm_cswap2(s1, s2);
        // class rows: s0 -> 0, s1 -> 1 (2 if diagonal), s2 -> 3 (4), s3 -> 5
        const uint32_t diag = ((((s0 ^ s1) & 0x00030003u) + K1) >> 2) & K1;  // 1 per half iff slots {0,3} / {1,2}
        if constexpr (BA) {
            constexpr uint32_t LM = 0xFFFCFFFCu;
            const uint32_t Sb = 4u * M2;  // row stride in bytes
            const uint32_t w[4] = {s0 & LM, (s1 & LM) + (K1 + diag) * Sb, (s2 & LM) + (3u * K1 + diag) * Sb,
                                   (s3 & LM) + 5u * Sb * K1};
#pragma unroll
            for (int e = 0; e < 4; ++e) sinc2(w[e], vsel, top);
        } else {
            const uint32_t i0 = (s0 >> 2) & 0x3FFF3FFFu;
            const uint32_t i1 = ((s1 >> 2) & 0x3FFF3FFFu) + (K1 + diag) * M2;
            const uint32_t i2 = ((s2 >> 2) & 0x3FFF3FFFu) + (3u * K1 + diag) * M2;
            const uint32_t i3 = ((s3 >> 2) & 0x3FFF3FFFu) + 5u * M2 * K1;
            const uint32_t w[4] = {i0, i1, i2, i3};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t x = (w[e] & vmask) | (dummy & ~vmask);
                ft_sh_add(h, x & 0xFFFFu, 7u * M2);
                ft_sh_add(h, x >> 16, 7u * M2);
            }
        }
        a = u0 - 2u * K1;
        c = u1 - 2u * K1;
    };

    P2 raw[HM_PF];
    {
        P2 r0;
        fetch(0, ptr, r0);
        const uint32_t V0 = t_lo <= 0 && 0 < t_hi ? quant_in(r0) : S;  // row ia-1
        const uint32_t Wm0 = shift_pair(__shfl_up_sync(FULL, V0, 1), V0);
        a = Wm0;            // NW (slot 0)
        c = V0 + K1;        // NE (slot 1)
        hm_cswap2(a, c);
    }
#pragma unroll
    for (int p = 0; p < HM_PF; ++p) fetch(p + 1, ptr + (p + 1) * g.W, raw[p]);
    ptr += (HM_PF + 1) * g.W;  // row t = PF+1
    const int nm = min(n, t_hi - 1);  // steps s < nm see an existing row t = s+1
    int s = 0;
    for (; s + HM_PF <= nm && s + 2 * HM_PF < tf; s += HM_PF) {
#pragma unroll
        for (int p = 0; p < HM_PF; ++p) {
            const uint32_t V = quant_in(raw[p]);
            raw[p] = load_pair<DT, VEC>(ptr + p * g.W, true, EDGE ? kk + 1 < Wi : true);
            step(V);
        }
        ptr += HM_PF * g.W;
    }
    for (; s < nm; s += HM_PF) {
#pragma unroll
        for (int p = 0; p < HM_PF; ++p) {
            if (s + p < nm) {
                const uint32_t V = quant_in(raw[p]);
                fetch(s + p + HM_PF + 1, ptr + p * g.W, raw[p]);
                step(V);
            }
        }
        ptr += HM_PF * g.W;
    }
    if (nm < n) step(S);  // vertex row H: the absent row below
}

template <int DT, int QM, bool VEC, bool BA>
__global__ void __launch_bounds__(HM_NTH, 2) hist2d_march(const typename Elem<DT>::T* __restrict__ buf, Geo2 g,
                                                         QuantDev q, unsigned long long* __restrict__ hist)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int M2 = g.M + 2;
    uint32_t* h = reinterpret_cast<uint32_t*>(smem_raw);  // 6 class rows + the dummy row
    float* tt = reinterpret_cast<float*>(h + 7 * M2);
    for (int i = threadIdx.x; i < 7 * M2; i += blockDim.x) h[i] = 0;
    if (QM != FT_Q_IDENTITY && QM != FT_Q_POW2)
        for (int i = threadIdx.x; i < M2; i += blockDim.x) tt[i] = q.tt[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t hb = (uint32_t)__cvta_generic_to_shared(h);
    constexpr int NW = HM_NTH / 32;
    const int64_t nrows = g.v1 - g.v0;
    const int ntiles = g.tiles;
    const int64_t Timg = cdiv(nrows, (int64_t)HM_RB) * ntiles * HM_RB;
    const int64_t total = g.batch * Timg;
    const int64_t U0 = total * blockIdx.x / gridDim.x, U1 = total * (blockIdx.x + 1) / gridDim.x;
    for (int64_t b = U0 / Timg; b < g.batch && b * Timg < U1; ++b) {
        const int64_t a = max(U0, b * Timg) - b * Timg, e = min(U1, (b + 1) * Timg) - b * Timg;
        const int64_t wa = a + (e - a) * warp / NW, we = a + (e - a) * (warp + 1) / NW;
        const typename Elem<DT>::T* img = buf + b * g.bstride;
        for (int64_t u = wa; u < we;) {
            const int64_t piece = u / HM_RB;
            const int r = (int)(u - piece * HM_RB);
            const int64_t len = min(we - u, (int64_t)(HM_RB - r));
            u += len;
            const int64_t rb = piece / ntiles;
            const int t = (int)(piece - rb * ntiles);
            const int64_t r0 = rb * HM_RB + r, r1 = min(r0 + len, nrows);
            if (r0 >= r1) continue;
            const int k0 = t * 62 - 1;
            if (k0 >= 1 && k0 + 63 <= g.W)
                hm_item<DT, QM, VEC, false, BA>(img, g, q, tt, h, hb, g.v0 + r0, g.v0 + r1, k0, lane);
            else
                hm_item<DT, QM, VEC, true, BA>(img, g, q, tt, h, hb, g.v0 + r0, g.v0 + r1, k0, lane);
        }
        __syncthreads();
        unsigned long long* out = hist + b * FT_NCLASS_2D * M2;
        for (int i = threadIdx.x; i < 7 * M2; i += blockDim.x) {
            const uint32_t v = h[i];
            h[i] = 0;
            // BA: bin (row r, level l) sits r M2 + l + 1 words below word 6 M2
            if (v && i < 6 * M2) atomicAdd(&out[BA ? 6 * M2 - 1 - i : i], (unsigned long long)v);
        }
        __syncthreads();
    }
}

static int sm_count2()
{
    int dev = 0, n = kSMs;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

template <int DT, int QM>
static int launch2(const ft_window* win, int64_t H, int64_t W, int64_t v0, int64_t v1, const ft_quant* qa,
                   int32_t M, uint64_t* hist, cudaStream_t st)
{
    using T = typename Elem<DT>::T;
    const T* buf = static_cast<const T*>(win->data);
    Geo2 g{};
    g.H = H; g.W = W; g.v0 = v0; g.v1 = v1; g.first = win->first; g.M = M;
    g.batch = std::max<int64_t>(win->batch, 1);
    g.bstride = win->batch_stride;
    QuantDev q{qa ? qa->mode : FT_Q_IDENTITY, qa ? qa->negate : 0, qa ? qa->scale : 0.f,
               qa ? qa->bias : 0.f, qa ? qa->thresholds : nullptr};
    const int M2 = M + 2;
    auto* out = reinterpret_cast<unsigned long long*>(hist);
    const int nsm = sm_count2();
    if (7 * M2 <= 0xFFFF && (size_t)8 * M2 * 4 <= 227 * 1024) {
        // register march: every vertex column 0..W
        const bool vec = W % 2 == 0 && (g.batch <= 1 || g.bstride % 2 == 0) &&
                         reinterpret_cast<uintptr_t>(buf) % (2 * sizeof(T)) == 0;
#ifdef HM2_NO_BA
        const bool ba = false;
#else
        const bool ba = 24 * M2 <= 0xFFFF;  // 6 rows of byte offsets in the 16-bit halves (M <= 2728)
#endif
        auto kern = ba ? (vec ? hist2d_march<DT, QM, true, true> : hist2d_march<DT, QM, false, true>)
                       : (vec ? hist2d_march<DT, QM, true, false> : hist2d_march<DT, QM, false, false>);
        const size_t sm = (size_t)8 * M2 * 4;
        FT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        int per_sm = 0;
        FT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, HM_NTH, sm));
        if (per_sm < 1) return FT_ERR_INTERNAL;
        g.tiles = (int)((W + 1) / 62 + 1);  // tile t: vertex columns 62 t - 1 .. 62 t + 60
        const int64_t units = g.batch * cdiv(v1 - v0, (int64_t)HM_RB) * g.tiles * HM_RB;
        const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)nsm * per_sm,
                                                                    cdiv(units, (int64_t)(HM_NTH / 32) * HM_RB)));
        kern<<<(int)grid, HM_NTH, sm, st>>>(buf, g, q, out);
        FT_CUDA_TRY(cudaGetLastError());
        return FT_OK;
    }
    const int64_t n = g.batch * (v1 - v0) * (W + 1);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), (int64_t)nsm * 8));
    constexpr int QW = QM == FT_Q_POW2 ? FT_Q_TABLE : QM;  // the table ships with FT_Q_POW2 too
    hist2d_wide<DT, QW><<<grid, 256, 0, st>>>(buf, g, q, out);
    FT_CUDA_TRY(cudaGetLastError());
    return FT_OK;
}

}  // namespace ft

using namespace ft;

extern "C" int ft_hist2d(const ft_window* win, int64_t H, int64_t W, int64_t v0, int64_t v1,
                         const ft_quant* q, int32_t M, uint64_t* hist, void* stream)
{
    if (!win || !hist || H < 1 || W < 1 || M < 0 || v0 < 0 || v1 > H + 1 || v0 > v1) return FT_ERR_ARG;
    if (win->batch > 1 && win->batch_stride < (int64_t)win->count * W) return FT_ERR_ARG;
    if (v0 == v1) return FT_OK;
    const int64_t need_lo = std::max<int64_t>(v0 - 1, 0), need_hi = std::min<int64_t>(v1 - 1, H - 1);
    if (need_lo <= need_hi && (win->data == nullptr || need_lo < win->first || need_hi >= win->first + win->count))
        return FT_ERR_ARG;
    if (M > (1 << 29) - 2) return FT_ERR_ARG;  // keys level*4 + slot in 32 bits
    const int qm = effective_qmode(q, true);  // FT_Q_POW2: table-free march quantizer
    if (qm != FT_Q_IDENTITY && !q->thresholds) return FT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (win->dtype) {
    case FT_I32:
        if (qm != FT_Q_IDENTITY) return FT_ERR_ARG;
        return launch2<FT_I32, FT_Q_IDENTITY>(win, H, W, v0, v1, q, M, hist, st);
    case FT_U8:
        if (qm == FT_Q_IDENTITY) return launch2<FT_U8, FT_Q_IDENTITY>(win, H, W, v0, v1, q, M, hist, st);
        if (qm == FT_Q_TABLE || qm == FT_Q_POW2) return launch2<FT_U8, FT_Q_TABLE>(win, H, W, v0, v1, q, M, hist, st);
        return launch2<FT_U8, FT_Q_TABLE_ROBUST>(win, H, W, v0, v1, q, M, hist, st);
    case FT_U16:
        if (qm == FT_Q_IDENTITY) return launch2<FT_U16, FT_Q_IDENTITY>(win, H, W, v0, v1, q, M, hist, st);
        if (qm == FT_Q_POW2) return launch2<FT_U16, FT_Q_POW2>(win, H, W, v0, v1, q, M, hist, st);
        if (qm == FT_Q_TABLE) return launch2<FT_U16, FT_Q_TABLE>(win, H, W, v0, v1, q, M, hist, st);
        return launch2<FT_U16, FT_Q_TABLE_ROBUST>(win, H, W, v0, v1, q, M, hist, st);
    case FT_F32:
        if (qm == FT_Q_IDENTITY) return FT_ERR_ARG;
        if (qm == FT_Q_POW2) return launch2<FT_F32, FT_Q_POW2>(win, H, W, v0, v1, q, M, hist, st);
        if (qm == FT_Q_TABLE) return launch2<FT_F32, FT_Q_TABLE>(win, H, W, v0, v1, q, M, hist, st);
        return launch2<FT_F32, FT_Q_TABLE_ROBUST>(win, H, W, v0, v1, q, M, hist, st);
    }
    return FT_ERR_ARG;
}
