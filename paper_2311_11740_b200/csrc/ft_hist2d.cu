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
// A CTA owns 256 vertex columns and marches rows: each step stages one cell
// row segment (+1 halo) as 16-bit levels (quantized on the fly); the row above
// stays in registers as a sorted pair, so a vertex sorts 2 new keys and
// merges (4 compare-exchanges).  Batches of equally-shaped images (config 3)
// run in one launch with one histogram per image.  The vertex column j == W
// is done by a flat kernel.
#include <algorithm>

#include "ft_common.cuh"
#include "ft_tables.h"

namespace ft {

constexpr int NT2 = 256;
constexpr int RW2 = NT2 + 1;  // staged cells per row segment
constexpr int PF2 = 2;

struct Geo2 {
    int64_t H, W, v0, v1, first, batch, bstride;
    int M;
    int tiles, chunk;
    int64_t n_items, items_per_image;
};

template <int DT, int QM>
__device__ __forceinline__ uint32_t level2(const typename Elem<DT>::T* __restrict__ img, const Geo2& g,
                                           int64_t r, int64_t c, const float* tt, const QuantDev& q)
{
    if (r < 0 || r >= g.H || c < 0 || c >= g.W) return (uint32_t)g.M + 1;
    return to_level<DT, QM>(ld_stream(img + (r - g.first) * g.W + c), tt, q.scale, q.bias, q.negate, g.M);
}

__device__ __forceinline__ void book2(uint32_t* __restrict__ h, uint32_t s0, uint32_t s1, uint32_t s2,
                                      uint32_t s3, int M2)
{
    const bool diag = ((s0 ^ s1) & 3) == 3;
    atomicAdd(&h[s0 >> 2], 1u);
    atomicAdd(&h[(diag ? 2 : 1) * M2 + (s1 >> 2)], 1u);
    atomicAdd(&h[(diag ? 4 : 3) * M2 + (s2 >> 2)], 1u);
    atomicAdd(&h[5 * M2 + (s3 >> 2)], 1u);
}

__device__ __forceinline__ void flush2(uint32_t* h, unsigned long long* __restrict__ out, int n, bool zero)
{
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        uint32_t v = h[i];
        if (v) atomicAdd(&out[i], (unsigned long long)v);
        if (zero) h[i] = 0;
    }
}

template <int DT, int QM>
__global__ void __launch_bounds__(NT2) hist2d_tiled(const typename Elem<DT>::T* __restrict__ buf, Geo2 g,
                                                    QuantDev q, unsigned long long* __restrict__ hist)
{
    using T = typename Elem<DT>::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int M2 = g.M + 2;
    const int NH = FT_NCLASS_2D * M2;
    uint32_t* h = reinterpret_cast<uint32_t*>(smem_raw);
    float* tt = reinterpret_cast<float*>(h + NH);
    uint16_t* rowbuf = reinterpret_cast<uint16_t*>(tt + M2);
    for (int i = threadIdx.x; i < NH; i += NT2) h[i] = 0;
    if (QM != FT_Q_IDENTITY)
        for (int i = threadIdx.x; i < M2; i += NT2) tt[i] = q.tt[i];
    __syncthreads();

    const int tid = threadIdx.x;
    const int64_t it0 = g.n_items * blockIdx.x / gridDim.x;
    const int64_t it1 = g.n_items * (blockIdx.x + 1) / gridDim.x;
    const uint32_t sentinel = (uint32_t)g.M + 1;
    int64_t cur_img = it0 < it1 ? it0 / g.items_per_image : 0;

    for (int64_t item = it0; item < it1; ++item) {
        const int64_t b = item / g.items_per_image;
        if (b != cur_img) {  // histogram belongs to one image: flush on change
            __syncthreads();
            flush2(h, hist + cur_img * NH, NH, true);
            __syncthreads();
            cur_img = b;
        }
        const int64_t rem = item - b * g.items_per_image;
        const int64_t ch = rem / g.tiles;
        const int64_t j0 = (rem % g.tiles) * NT2;
        const int64_t ia = g.v0 + ch * g.chunk;
        const int64_t ib = min(ia + (int64_t)g.chunk, g.v1);
        const T* img = buf + b * g.bstride;
        const bool active = j0 + tid < g.W;

        // cells (r, j0 - 1 + tid) and, for tid == 0, (r, j0 + 255)
        auto inside = [&](int64_t r, int e) {
            const int64_t c = e == 0 ? j0 - 1 + tid : j0 - 1 + NT2;
            return (e == 0 || tid == 0) && r >= 0 && r < g.H && c >= 0 && c < g.W;
        };
        T lv[PF2 + 1][2];
        auto fetch = [&](int64_t r, T (&dst)[2]) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                dst[e] = T(0);
                if (inside(r, e)) dst[e] = ld_stream(img + (r - g.first) * g.W + (e == 0 ? j0 - 1 + tid : j0 - 1 + NT2));
            }
        };
        auto store = [&](int64_t r, uint16_t* dst, const T (&src)[2]) {
            dst[tid] = (uint16_t)(inside(r, 0) ? to_level<DT, QM>(src[0], tt, q.scale, q.bias, q.negate, g.M) : sentinel);
            if (tid == 0)
                dst[NT2] = (uint16_t)(inside(r, 1) ? to_level<DT, QM>(src[1], tt, q.scale, q.bias, q.negate, g.M)
                                                   : sentinel);
        };
        fetch(ia - 1, lv[0]);
#pragma unroll
        for (int s = 1; s <= PF2; ++s) fetch(ia - 1 + s, lv[s]);
        store(ia - 1, rowbuf, lv[0]);
        __syncthreads();
        uint32_t a = (uint32_t)rowbuf[tid] * 4 + 0;
        uint32_t c = (uint32_t)rowbuf[tid + 1] * 4 + 1;
        cswap(a, c);

        for (int64_t i = ia; i < ib; ++i) {
            uint16_t* cur = rowbuf + ((i - ia + 1) & 1) * RW2;
            store(i, cur, lv[1]);
#pragma unroll
            for (int s = 1; s < PF2; ++s) {
                lv[s][0] = lv[s + 1][0];
                lv[s][1] = lv[s + 1][1];
            }
            if (i + PF2 < ib) fetch(i + PF2, lv[PF2]);
            __syncthreads();
            uint32_t u0 = (uint32_t)cur[tid] * 4 + 2;
            uint32_t u1 = (uint32_t)cur[tid + 1] * 4 + 3;
            cswap(u0, u1);
            if (active) {
                uint32_t s0 = a, s1 = c, s2 = u0, s3 = u1;
                merge22(s0, s1, s2, s3);
                book2(h, s0, s1, s2, s3, M2);
            }
            a = u0 - 2;
            c = u1 - 2;
        }
        __syncthreads();
    }
    __syncthreads();
    if (it0 < it1) flush2(h, hist + cur_img * NH, NH, false);
}

// Vertex column j == W of every vertex row in [v0, v1), all images.
template <int DT, int QM>
__global__ void __launch_bounds__(256) hist2d_edge(const typename Elem<DT>::T* __restrict__ buf, Geo2 g,
                                                   QuantDev q, unsigned long long* __restrict__ hist)
{
    const int M2 = g.M + 2;
    const int64_t n = g.batch * (g.v1 - g.v0);
    __shared__ float tt_s[1];  // thresholds read straight from global here
    (void)tt_s;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / (g.v1 - g.v0);
        const int64_t i = g.v0 + t % (g.v1 - g.v0);
        const auto* img = buf + b * g.bstride;
        const int64_t j = g.W;
        uint32_t k0 = level2<DT, QM>(img, g, i - 1, j - 1, q.tt, q) * 4 + 0;
        uint32_t k1 = level2<DT, QM>(img, g, i - 1, j, q.tt, q) * 4 + 1;
        uint32_t k2 = level2<DT, QM>(img, g, i, j - 1, q.tt, q) * 4 + 2;
        uint32_t k3 = level2<DT, QM>(img, g, i, j, q.tt, q) * 4 + 3;
        sort4(k0, k1, k2, k3);
        unsigned long long* hb = hist + b * (int64_t)FT_NCLASS_2D * M2;
        const bool diag = ((k0 ^ k1) & 3) == 3;
        atomicAdd(&hb[k0 >> 2], 1ull);
        atomicAdd(&hb[(diag ? 2 : 1) * M2 + (k1 >> 2)], 1ull);
        atomicAdd(&hb[(diag ? 4 : 3) * M2 + (k2 >> 2)], 1ull);
        atomicAdd(&hb[5 * M2 + (k3 >> 2)], 1ull);
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
    const size_t smem = (size_t)(FT_NCLASS_2D * M2 + M2) * 4 + 2 * RW2 * sizeof(uint16_t);
    auto* out = reinterpret_cast<unsigned long long*>(hist);
    const int nsm = sm_count2();
    {
        auto kern = hist2d_tiled<DT, QM>;
        FT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        FT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT2, smem));
        if (per_sm < 1) return FT_ERR_ARG;
        g.tiles = (int)cdiv(W, NT2);
        const int64_t rows = v1 - v0;
        const int64_t grid_cap = (int64_t)nsm * per_sm;
        const int64_t tiles_all = g.tiles * g.batch;
        int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>(cdiv(4 * grid_cap, tiles_all), rows / 64));
        g.chunk = (int)cdiv(rows, nchunks);
        nchunks = cdiv(rows, g.chunk);
        g.items_per_image = g.tiles * nchunks;
        g.n_items = g.items_per_image * g.batch;
        const int grid = (int)std::min<int64_t>(grid_cap, g.n_items);
        kern<<<grid, NT2, smem, st>>>(buf, g, q, out);
        FT_CUDA_TRY(cudaGetLastError());
    }
    {
        const int64_t n = g.batch * (v1 - v0);
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 4 * nsm));
        hist2d_edge<DT, QM><<<grid, 256, 0, st>>>(buf, g, q, out);
        FT_CUDA_TRY(cudaGetLastError());
    }
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
    const size_t smem = (size_t)(FT_NCLASS_2D * (M + 2) + (M + 2)) * 4 + 2 * RW2 * 2;
    if (smem > 227 * 1024 || M + 1 > 65535) return FT_ERR_ARG;
    const int qm = effective_qmode(q);
    if (qm != FT_Q_IDENTITY && !q->thresholds) return FT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (win->dtype) {
    case FT_I32:
        if (qm != FT_Q_IDENTITY) return FT_ERR_ARG;
        return launch2<FT_I32, FT_Q_IDENTITY>(win, H, W, v0, v1, q, M, hist, st);
    case FT_U8:
        if (qm == FT_Q_IDENTITY) return launch2<FT_U8, FT_Q_IDENTITY>(win, H, W, v0, v1, q, M, hist, st);
        if (qm == FT_Q_TABLE) return launch2<FT_U8, FT_Q_TABLE>(win, H, W, v0, v1, q, M, hist, st);
        return launch2<FT_U8, FT_Q_TABLE_ROBUST>(win, H, W, v0, v1, q, M, hist, st);
    case FT_U16:
        if (qm == FT_Q_IDENTITY) return launch2<FT_U16, FT_Q_IDENTITY>(win, H, W, v0, v1, q, M, hist, st);
        if (qm == FT_Q_TABLE) return launch2<FT_U16, FT_Q_TABLE>(win, H, W, v0, v1, q, M, hist, st);
        return launch2<FT_U16, FT_Q_TABLE_ROBUST>(win, H, W, v0, v1, q, M, hist, st);
    case FT_F32:
        if (qm == FT_Q_IDENTITY) return FT_ERR_ARG;
        if (qm == FT_Q_TABLE) return launch2<FT_F32, FT_Q_TABLE>(win, H, W, v0, v1, q, M, hist, st);
        return launch2<FT_F32, FT_Q_TABLE_ROBUST>(win, H, W, v0, v1, q, M, hist, st);
    }
    return FT_ERR_ARG;
}
