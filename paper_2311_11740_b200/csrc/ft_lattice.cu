// ft_lattice.cu -- fused descriptor histograms by lattice min/max filters.
//
// The curve path of the north star: "evaluate each vertex's integer EC and
// measure contributions into a filtration-level histogram, then a device
// prefix scan".  Instead of classifying sorted neighbourhoods, count the
// cells of the closed cubical complex by the level at which they appear:
// an element (face, edge, vertex) of the complex appears at the MIN level of
// its incident cells, so
//   EC_26C = V - E + F - C,  surface area = 2 F - 6 C,  volume = C     (3D)
//   EC_8C = V - E + C,  EC_4C = C - E_max + V_max,  perimeter = 2E - 4C,
//   area = C                                                           (2D)
// with V/E/F/C counted by level (E_max/V_max: all incident cells active =
// MAX filters).  These are the reference's vertex-contribution curves
// (descriptors.py:169-178 over contrib2d/3d maps) rewritten; tests pin them
// to the reference golden curves.  No tie-breaking enters: min/max are
// order-free, so the curves are bit-exact without sorting.
//
// Every lattice point p = (i, j, k) owns its low-corner vertex, the three
// edges and three faces leaving it in + directions... equivalently the
// elements whose incident cells are c - {0,1}^S (c = cell (i,j,k)).  Per
// point: 3 face mins, 3 edge mins, 1 vertex min (7 VIMNMX on 16-bit pairs:
// two lattice points per instruction) and 8 shared-memory increments into 4
// histograms [cells, faces, edges, vertices].  Absent cells carry the
// sentinel M+1 (elements touching only absent cells land in bin M+1, which
// no curve reads), so tiles simply pad with sentinels: no boundary kernel.
//
// Layout: levels are staged as 16-bit (level * 4) in shared memory, two
// k-adjacent cells per 32-bit word, so packed mins and the per-event
// byte-address extraction are one instruction each.
#include <algorithm>

#include "ft_common.cuh"
#include "ft_tables.h"

namespace ft {

constexpr int LTW = 32;                 // words (2 lattice points) per tile row = one warp
constexpr int LTJ = 16;                 // tile rows (warps)
constexpr int LNT = LTW * LTJ;          // 512 threads
constexpr int LPW = LTW + 1;            // staged words per row (one halo word on the low side)
constexpr int LPN = (LTJ + 1) * LPW;    // staged words per plane
constexpr int LLD = (LPN + LNT - 1) / LNT;
constexpr int LPF = 2;                  // planes in flight

struct LGeo {
    int64_t H, W, D, v0, v1, first, bstride;
    int M, tiles_j, tiles_k, chunk;
    int64_t n_items, items_per_image;
};

__device__ __forceinline__ uint32_t vmin2(uint32_t a, uint32_t b) { return __vminu2(a, b); }
__device__ __forceinline__ uint32_t vmax2(uint32_t a, uint32_t b) { return __vmaxu2(a, b); }
// (hi half of a, lo half of b): the pair shifted down by one cell
__device__ __forceinline__ uint32_t shift_pair(uint32_t a, uint32_t b) { return __byte_perm(a, b, 0x5432); }

__device__ __forceinline__ void inc2(uint32_t* __restrict__ h, uint32_t w)
{
    // w holds two byte offsets (level * 4) of two lattice points
    atomicAdd(reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(h) + (w & 0xFFFFu)), 1u);
    atomicAdd(reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(h) + (w >> 16)), 1u);
}

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

template <int DT, int QM>
__device__ __forceinline__ uint32_t pack_pair(const typename Pair<DT>::T& v, bool okx, bool oky, const float* tt,
                                              const QuantDev& q, int M, uint32_t sent4)
{
    const uint32_t a = okx ? to_level4<DT, QM>(v.x, tt, q.scale, q.bias, q.negate, M) : sent4;
    const uint32_t b = oky ? to_level4<DT, QM>(v.y, tt, q.scale, q.bias, q.negate, M) : sent4;
    return __byte_perm(a, b, 0x5410);
}

// ------------------------------------------------------------------- 3D

template <int DT, int QM, bool VEC>
__global__ void __launch_bounds__(LNT) lattice3d_kernel(const typename Elem<DT>::T* __restrict__ buf, LGeo g,
                                                         QuantDev q, unsigned long long* __restrict__ hist)
{
    using P2 = typename Pair<DT>::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int M2 = g.M + 2;
    uint32_t* h = reinterpret_cast<uint32_t*>(smem_raw);  // [4][M2]: cells, faces, edges, vertices
    float* tt = reinterpret_cast<float*>(h + 4 * M2);
    uint32_t* pl = reinterpret_cast<uint32_t*>(tt + M2);  // [2][LPN] words
    for (int i = threadIdx.x; i < 4 * M2; i += LNT) h[i] = 0;
    if (QM != FT_Q_IDENTITY)
        for (int i = threadIdx.x; i < M2; i += LNT) tt[i] = q.tt[i];
    __syncthreads();
    uint32_t* hv = h;
    uint32_t* hf = h + M2;
    uint32_t* he = h + 2 * M2;
    uint32_t* hx = h + 3 * M2;

    const int tid = threadIdx.x;
    const int ty = tid / LTW, tx = tid % LTW;
    const int Wi = (int)g.W, Di = (int)g.D;
    const int64_t plane_elems = g.W * g.D;
    const uint32_t sent2 = ((uint32_t)(g.M + 1) * 4u) * 0x10001u;
    const int64_t per_chunk = (int64_t)g.tiles_j * g.tiles_k;
    const int64_t it0 = g.n_items * blockIdx.x / gridDim.x;
    const int64_t it1 = g.n_items * (blockIdx.x + 1) / gridDim.x;

    int lr[LLD], lw[LLD];
#pragma unroll
    for (int e = 0; e < LLD; ++e) {
        const int idx = tid + e * LNT;
        lr[e] = idx / LPW;
        lw[e] = idx % LPW;
    }

    for (int64_t item = it0; item < it1; ++item) {
        const int64_t ch = item / per_chunk;
        const int rem = (int)(item - ch * per_chunk);
        const int j0 = (rem / g.tiles_k) * LTJ;
        const int k0 = (rem % g.tiles_k) * (2 * LTW);
        const int64_t ia = g.v0 + ch * g.chunk;
        const int64_t ib = min(ia + (int64_t)g.chunk, g.v1);

        // staged word (r, w) = cells (row j0-1+r, cols k0-2+2w and +1)
        int off[LLD];
        bool okx[LLD], oky[LLD];
#pragma unroll
        for (int e = 0; e < LLD; ++e) {
            const int jj = j0 - 1 + lr[e], kk = k0 - 2 + 2 * lw[e];
            const bool row = (tid + e * LNT < LPN) && jj >= 0 && jj < Wi && kk >= 0;
            okx[e] = row && kk < Di;
            oky[e] = row && kk + 1 < Di;
            off[e] = okx[e] ? jj * Di + kk : 0;
        }
        auto fetch = [&](int64_t p, P2 (&dst)[LLD]) {
            const bool pin = p >= 0 && p < g.H;
            const typename Elem<DT>::T* base = buf + (pin ? (p - g.first) * plane_elems : 0);
#pragma unroll
            for (int e = 0; e < LLD; ++e) dst[e] = load_pair<DT, VEC>(base + off[e], pin && okx[e], pin && oky[e]);
        };
        const uint32_t sent4 = (uint32_t)(g.M + 1) * 4u;
        auto store = [&](int64_t p, uint32_t* dstp, const P2 (&src)[LLD]) {
            const bool pin = p >= 0 && p < g.H;
#pragma unroll
            for (int e = 0; e < LLD; ++e) {
                const int idx = tid + e * LNT;
                if (idx < LPN) dstp[idx] = pack_pair<DT, QM>(src[e], pin && okx[e], pin && oky[e], tt, q, g.M, sent4);
            }
        };
        // raw ring without register moves: ra holds the next even step's
        // plane, rb the next odd step's; each is refilled right after use
        P2 ra[LLD], rb[LLD];
        fetch(ia - 1, ra);
        store(ia - 1, pl, ra);
        fetch(ia, ra);
        fetch(ia + 1, rb);
        __syncthreads();

        // thread = lattice points (j0+ty, k0+2tx .. +1): cur row word cw
        const int cw = (ty + 1) * LPW + tx + 1;
        uint32_t W_ = pl[cw], U = pl[cw - LPW];
        uint32_t Wm = shift_pair(pl[cw - 1], W_), Um = shift_pair(pl[cw - LPW - 1], U);
        uint32_t pW = W_;
        uint32_t pm2k = vmin2(W_, Wm);
        uint32_t pm2j = vmin2(W_, U);
        uint32_t pm4i = vmin2(pm2k, vmin2(U, Um));

        auto step = [&](const uint32_t* cur) {
            W_ = cur[cw];
            U = cur[cw - LPW];
            Wm = shift_pair(cur[cw - 1], W_);
            Um = shift_pair(cur[cw - LPW - 1], U);
            const uint32_t m2k = vmin2(W_, Wm);             // face normal k
            const uint32_t m2j = vmin2(W_, U);              // face normal j
            const uint32_t m4i = vmin2(m2k, vmin2(U, Um));  // edge along i
            inc2(hv, W_);
            inc2(hf, vmin2(W_, pW));     // face normal i
            inc2(hf, m2j);
            inc2(hf, m2k);
            inc2(he, m4i);
            inc2(he, vmin2(m2k, pm2k));  // edge along j
            inc2(he, vmin2(m2j, pm2j));  // edge along k
            inc2(hx, vmin2(m4i, pm4i));  // vertex
            pW = W_;
            pm2k = m2k;
            pm2j = m2j;
            pm4i = m4i;
        };
        for (int64_t i = ia; i < ib; i += 2) {
            uint32_t* cur = pl + LPN;  // plane i (i - ia even) -> buffer 1
            store(i, cur, ra);
            if (i + 2 < ib) fetch(i + 2, ra);
            __syncthreads();
            step(cur);
            if (i + 1 >= ib) break;
            cur = pl;                  // plane i + 1 -> buffer 0
            store(i + 1, cur, rb);
            if (i + 3 < ib) fetch(i + 3, rb);
            __syncthreads();
            step(cur);
        }
        __syncthreads();
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4 * M2; i += LNT) {
        const uint32_t v = h[i];
        if (v) atomicAdd(&hist[i], (unsigned long long)v);
    }
}

// ------------------------------------------------------------------- 2D
// Lattice point p = (i, j) owns its low-corner vertex (cells (i-1..i,
// j-1..j)), the edge to (i, j+1) (cells (i-1, j), (i, j)), the edge to
// (i+1, j) (cells (i, j-1), (i, j)) and the cell (i, j).  Rows: cells, edge
// mins, vertex maxes (the last only for EC_4C; E_max = 4C - E is implied).
constexpr int L2W = 256;                 // words per row segment (512 lattice columns)
constexpr int L2N = L2W + 1;

template <int DT, int QM, bool MAXES, bool VEC>
__global__ void __launch_bounds__(L2W) lattice2d_kernel(const typename Elem<DT>::T* __restrict__ buf, LGeo g,
                                                         QuantDev q, unsigned long long* __restrict__ hist)
{
    using P2 = typename Pair<DT>::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int M2 = g.M + 2;
    constexpr int NR = 4;
    uint32_t* h = reinterpret_cast<uint32_t*>(smem_raw);
    float* tt = reinterpret_cast<float*>(h + NR * M2);
    uint32_t* rows = reinterpret_cast<uint32_t*>(tt + M2);  // [2][L2N]
    for (int i = threadIdx.x; i < NR * M2; i += L2W) h[i] = 0;
    if (QM != FT_Q_IDENTITY)
        for (int i = threadIdx.x; i < M2; i += L2W) tt[i] = q.tt[i];
    __syncthreads();
    uint32_t *hc = h, *he = h + M2, *hx = h + 2 * M2, *hX = h + 3 * M2;

    const int tid = threadIdx.x;
    const uint32_t sent2 = ((uint32_t)(g.M + 1) * 4u) * 0x10001u;
    const int Wi = (int)g.W;
    const int64_t it0 = g.n_items * blockIdx.x / gridDim.x;
    const int64_t it1 = g.n_items * (blockIdx.x + 1) / gridDim.x;
    int64_t cur_img = it0 < it1 ? it0 / g.items_per_image : 0;

    for (int64_t item = it0; item < it1; ++item) {
        const int64_t b = item / g.items_per_image;
        if (b != cur_img) {
            __syncthreads();
            for (int i = threadIdx.x; i < NR * M2; i += L2W) {
                const uint32_t v = h[i];
                if (v) atomicAdd(&hist[cur_img * NR * M2 + i], (unsigned long long)v);
                h[i] = 0;
            }
            __syncthreads();
            cur_img = b;
        }
        const int64_t rem = item - b * g.items_per_image;
        const int64_t ch = rem / g.tiles_k;
        const int j0 = (int)(rem % g.tiles_k) * (2 * L2W);
        const int64_t ia = g.v0 + ch * g.chunk;
        const int64_t ib = min(ia + (int64_t)g.chunk, g.v1);
        const typename Elem<DT>::T* img = buf + b * g.bstride;
        // staged word w = cells (j0-2+2w, +1); thread tid owns word tid+1,
        // thread 0 also loads word 0
        const int kk0 = j0 - 2 + 2 * (tid + 1), kk1 = j0 - 2;
        const bool ok0x = kk0 >= 0 && kk0 < Wi, ok0y = kk0 >= 0 && kk0 + 1 < Wi;
        const bool ok1x = (tid == 0) && kk1 >= 0 && kk1 < Wi, ok1y = (tid == 0) && kk1 >= 0 && kk1 + 1 < Wi;
        const uint32_t sent4 = (uint32_t)(g.M + 1) * 4u;
        P2 raw[LPF + 1][2];
        auto fetch = [&](int64_t r, P2 (&dst)[2]) {
            const bool rin = r >= 0 && r < g.H;
            const auto* base = img + (rin ? (r - g.first) * g.W : 0);
            dst[0] = load_pair<DT, VEC>(base + (ok0x ? kk0 : 0), rin && ok0x, rin && ok0y);
            dst[1] = load_pair<DT, VEC>(base + (ok1x ? kk1 : 0), rin && ok1x, rin && ok1y);
        };
        auto store = [&](int64_t r, uint32_t* dst, const P2 (&src)[2]) {
            const bool rin = r >= 0 && r < g.H;
            dst[tid + 1] = pack_pair<DT, QM>(src[0], rin && ok0x, rin && ok0y, tt, q, g.M, sent4);
            if (tid == 0) dst[0] = pack_pair<DT, QM>(src[1], rin && ok1x, rin && ok1y, tt, q, g.M, sent4);
        };
        fetch(ia - 1, raw[0]);
#pragma unroll
        for (int s = 1; s <= LPF; ++s) fetch(ia - 1 + s, raw[s]);
        store(ia - 1, rows, raw[0]);
        __syncthreads();
        uint32_t pW = rows[tid + 1];
        uint32_t pWm = shift_pair(rows[tid], pW);
        for (int64_t i = ia; i < ib; ++i) {
            uint32_t* cur = rows + ((i - ia + 1) & 1) * L2N;
            store(i, cur, raw[1]);
#pragma unroll
            for (int s = 1; s < LPF; ++s) {
                raw[s][0] = raw[s + 1][0];
                raw[s][1] = raw[s + 1][1];
            }
            if (i + LPF < ib) fetch(i + LPF, raw[LPF]);
            __syncthreads();
            const uint32_t W_ = cur[tid + 1];
            const uint32_t Wm = shift_pair(cur[tid], W_);
            const uint32_t eh = vmin2(W_, pW);            // edge (i,j)-(i,j+1): cells (i-1,j), (i,j)
            const uint32_t ev = vmin2(W_, Wm);            // edge (i,j)-(i+1,j): cells (i,j-1), (i,j)
            inc2(hc, W_);
            inc2(he, eh);
            inc2(he, ev);
            inc2(hx, vmin2(ev, vmin2(pW, pWm)));
            if constexpr (MAXES) {
                inc2(hX, vmax2(vmax2(W_, Wm), vmax2(pW, pWm)));
            }
            pW = W_;
            pWm = Wm;
        }
        __syncthreads();
    }
    __syncthreads();
    if (it0 < it1)
        for (int i = threadIdx.x; i < NR * M2; i += L2W) {
            const uint32_t v = h[i];
            if (v) atomicAdd(&hist[cur_img * NR * M2 + i], (unsigned long long)v);
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
                    qa ? qa->thresholds : nullptr};
}

template <int DT, int QM>
static int launch_l3(const ft_window* win, int64_t H, int64_t W, int64_t D, int64_t v0, int64_t v1,
                     const ft_quant* qa, int32_t M, uint64_t* hist, cudaStream_t st)
{
    LGeo g{};
    g.H = H; g.W = W; g.D = D; g.v0 = v0; g.v1 = v1; g.first = win->first; g.M = M;
    const size_t smem = (size_t)(5 * (M + 2)) * 4 + 2 * LPN * 4;
    auto kern = (D % 2 == 0 && reinterpret_cast<uintptr_t>(win->data) % 8 == 0) ? lattice3d_kernel<DT, QM, true>
                                                                                 : lattice3d_kernel<DT, QM, false>;
    FT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    FT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, LNT, smem));
    if (per_sm < 1) return FT_ERR_ARG;
    // lattice points j in [0, W], k in [0, D] (the high boundary included)
    g.tiles_j = (int)cdiv(W + 1, LTJ);
    g.tiles_k = (int)cdiv(D + 1, 2 * LTW);
    const int64_t tiles = (int64_t)g.tiles_j * g.tiles_k;
    const int64_t rows = v1 - v0;
    const int64_t grid_cap = (int64_t)nsm_l() * per_sm;
    int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>(cdiv(6 * grid_cap, tiles), rows / 32));
    g.chunk = (int)cdiv(rows, nchunks);
    nchunks = cdiv(rows, g.chunk);
    g.n_items = tiles * nchunks;
    const int grid = (int)std::min<int64_t>(grid_cap, g.n_items);
    kern<<<grid, LNT, smem, st>>>(static_cast<const typename Elem<DT>::T*>(win->data), g, qdev(qa),
                                  reinterpret_cast<unsigned long long*>(hist));
    FT_CUDA_TRY(cudaGetLastError());
    return FT_OK;
}

template <int DT, int QM>
static int launch_l2(const ft_window* win, int64_t H, int64_t W, int64_t v0, int64_t v1, const ft_quant* qa,
                     int32_t M, int maxes, uint64_t* hist, cudaStream_t st)
{
    LGeo g{};
    g.H = H; g.W = W; g.D = 1; g.v0 = v0; g.v1 = v1; g.first = win->first; g.M = M;
    g.bstride = win->batch_stride;
    const int64_t batch = std::max<int64_t>(win->batch, 1);
    const size_t smem = (size_t)(5 * (M + 2)) * 4 + 2 * L2N * 4;
    const bool vec = W % 2 == 0 && (win->batch <= 1 || win->batch_stride % 2 == 0) &&
                     reinterpret_cast<uintptr_t>(win->data) % 8 == 0;
    auto kern = maxes ? (vec ? lattice2d_kernel<DT, QM, true, true> : lattice2d_kernel<DT, QM, true, false>)
                      : (vec ? lattice2d_kernel<DT, QM, false, true> : lattice2d_kernel<DT, QM, false, false>);
    FT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    FT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, L2W, smem));
    if (per_sm < 1) return FT_ERR_ARG;
    g.tiles_k = (int)cdiv(W + 1, 2 * L2W);
    const int64_t rows = v1 - v0;
    const int64_t grid_cap = (int64_t)nsm_l() * per_sm;
    const int64_t tiles_all = (int64_t)g.tiles_k * batch;
    int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>(cdiv(4 * grid_cap, tiles_all), rows / 64));
    g.chunk = (int)cdiv(rows, nchunks);
    nchunks = cdiv(rows, g.chunk);
    g.items_per_image = g.tiles_k * nchunks;
    g.n_items = g.items_per_image * batch;
    const int grid = (int)std::min<int64_t>(grid_cap, g.n_items);
    kern<<<grid, L2W, smem, st>>>(static_cast<const typename Elem<DT>::T*>(win->data), g, qdev(qa),
                                  reinterpret_cast<unsigned long long*>(hist));
    FT_CUDA_TRY(cudaGetLastError());
    return FT_OK;
}

static bool window_ok(const ft_window* win, int64_t H, int64_t v0, int64_t v1)
{
    const int64_t need_lo = std::max<int64_t>(v0 - 1, 0), need_hi = std::min<int64_t>(v1 - 1, H - 1);
    return !(need_lo <= need_hi &&
             (win->data == nullptr || need_lo < win->first || need_hi >= win->first + win->count));
}

}  // namespace ft

using namespace ft;

#define FT_LDISPATCH(LAUNCH, ...)                                                          \
    switch (win->dtype) {                                                                  \
    case FT_I32:                                                                           \
        if (qm != FT_Q_IDENTITY) return FT_ERR_ARG;                                        \
        return LAUNCH<FT_I32, FT_Q_IDENTITY>(__VA_ARGS__);                                 \
    case FT_U8:                                                                            \
        if (qm == FT_Q_IDENTITY) return LAUNCH<FT_U8, FT_Q_IDENTITY>(__VA_ARGS__);         \
        if (qm == FT_Q_TABLE) return LAUNCH<FT_U8, FT_Q_TABLE>(__VA_ARGS__);               \
        return LAUNCH<FT_U8, FT_Q_TABLE_ROBUST>(__VA_ARGS__);                              \
    case FT_U16:                                                                           \
        if (qm == FT_Q_IDENTITY) return LAUNCH<FT_U16, FT_Q_IDENTITY>(__VA_ARGS__);        \
        if (qm == FT_Q_TABLE) return LAUNCH<FT_U16, FT_Q_TABLE>(__VA_ARGS__);              \
        return LAUNCH<FT_U16, FT_Q_TABLE_ROBUST>(__VA_ARGS__);                             \
    case FT_F32:                                                                           \
        if (qm == FT_Q_IDENTITY) return FT_ERR_ARG;                                        \
        if (qm == FT_Q_TABLE) return LAUNCH<FT_F32, FT_Q_TABLE>(__VA_ARGS__);              \
        return LAUNCH<FT_F32, FT_Q_TABLE_ROBUST>(__VA_ARGS__);                             \
    }                                                                                      \
    return FT_ERR_ARG;

extern "C" int ft_lattice3d(const ft_window* win, int64_t H, int64_t W, int64_t D, int64_t v0, int64_t v1,
                            const ft_quant* q, int32_t M, uint64_t* hist, void* stream)
{
    if (!win || !hist || H < 1 || W < 1 || D < 1 || M < 0 || v0 < 0 || v1 > H + 1 || v0 > v1) return FT_ERR_ARG;
    if (W * D > INT32_MAX / 2 || (M + 1) * 4 > 0xFFFF) return FT_ERR_ARG;
    if (v0 == v1) return FT_OK;
    if (!window_ok(win, H, v0, v1)) return FT_ERR_ARG;
    const int qm = effective_qmode(q);
    if (qm != FT_Q_IDENTITY && !q->thresholds) return FT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    FT_LDISPATCH(launch_l3, win, H, W, D, v0, v1, q, M, hist, st)
}

extern "C" int ft_lattice2d(const ft_window* win, int64_t H, int64_t W, int64_t v0, int64_t v1,
                            const ft_quant* q, int32_t M, int32_t maxes, uint64_t* hist, void* stream)
{
    if (!win || !hist || H < 1 || W < 1 || M < 0 || v0 < 0 || v1 > H + 1 || v0 > v1) return FT_ERR_ARG;
    if ((M + 1) * 4 > 0xFFFF) return FT_ERR_ARG;
    if (win->batch > 1 && win->batch_stride < win->count * W) return FT_ERR_ARG;
    if (v0 == v1) return FT_OK;
    if (!window_ok(win, H, v0, v1)) return FT_ERR_ARG;
    const int qm = effective_qmode(q);
    if (qm != FT_Q_IDENTITY && !q->thresholds) return FT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    FT_LDISPATCH(launch_l2, win, H, W, v0, v1, q, M, maxes, hist, st)
}
