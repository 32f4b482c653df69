// ft_lattice.cu -- fused descriptor histograms by lattice min/max filters.
//
// The curve path of the north star: "evaluate each vertex's integer EC and
// measure contributions into a filtration-level histogram, then a device
// prefix scan".  Instead of classifying sorted neighbourhoods, count the
// cells of the closed cubical complex by the level at which they appear: an
// element (face, edge, vertex) appears at the MIN level of its incident cells,
// so
//   EC_26C = V - E + F - C,  surface area = 2F - 6C,  volume = C      (3D)
//   EC_8C = V - E + C,  EC_4C = -3C + E + V_max,  perimeter = 2E - 4C,
//   area = C                                                           (2D)
// with V/E/F/C counted by level (V_max: all incident cells active = MAX
// filter).  These are the reference's vertex-contribution curves
// (descriptors.py:169-178 over contrib2d/3d maps) rewritten (lattice.py holds
// the algebra; tests pin it to the reference golden curves).  No tie-breaking
// enters -- min/max are order-free -- so the curves are bit-exact without a
// sort.
//
// Every lattice point p = (i, j, k) owns the elements whose incident cells
// are c - {0,1}^S, c = cell (i, j, k): the cube, three faces, three edges and
// the vertex.  Per point: 7 packed 16-bit mins (two points per VIMNMX) and 8
// shared-memory increments into 4 histograms.  Absent cells carry the
// sentinel M+1 (elements touching only absent cells land in bin M+1, which no
// curve reads), so tiles pad with sentinels and need no boundary kernel.
//
// Layout (3D): a 512-thread CTA stages a 16 x 32-word plane tile per step,
// one word (two k-adjacent cells, levels * 4 as 16-bit lanes) per thread, and
// 15 x 31 threads compute 15 lattice rows x 62 lattice columns from it (row
// 0 / word 0 are the low halo).  One global load per thread per plane keeps
// the warps balanced at the per-plane barrier.  Each event is one LOP/LEA
// (extract a 16-bit byte offset) + one ATOMS on a uniform row base; the
// histograms are privatised per lane group to keep those ATOMS bank-conflict
// free (see Priv below).
#include "ft_lattice.cuh"
#include "ft_tables.h"

namespace ft {


// ------------------------------------------------------------------- 3D

template <int DT, int QM, bool VEC, int CP>
__global__ void __launch_bounds__(LNT) lattice3d_kernel(const typename Elem<DT>::T* __restrict__ buf, LGeo g,
                                                         QuantDev q, unsigned long long* __restrict__ hist)
{
    using P2 = typename Pair<DT>::T;
    using T = typename Elem<DT>::T;
    constexpr int SH = Priv<CP>::SH;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int M2 = g.M + 2;
    const int hs = g.hs;                                  // bytes between histogram rows
    char* h = reinterpret_cast<char*>(smem_raw);          // rows: cells, faces, edges, vertices
    float* tt = reinterpret_cast<float*>(h + 4 * hs);
    uint32_t* pl = reinterpret_cast<uint32_t*>(tt + M2);  // [2][LNT] staged words
    for (int i = threadIdx.x; i < hs; i += LNT) reinterpret_cast<uint32_t*>(h)[i] = 0;  // 4 rows = hs words
    if (QM != FT_Q_IDENTITY)
        for (int i = threadIdx.x; i < M2; i += LNT) tt[i] = q.tt[i];
    __syncthreads();

    const int tid = threadIdx.x;
    const int ty = tid / LTW, tx = tid % LTW;
    const bool computes = ty < LCJ && tx < LCW;
    const int Wi = (int)g.W, Di = (int)g.D;
    const int64_t plane_elems = g.W * g.D;
    const uint32_t sent4 = ((uint32_t)(g.M + 1) * 4u) << SH;
    const uint32_t cpy = (uint32_t)(tid % CP) * 4u * 0x10001u;  // this lane's histogram copy, both halves
    const int64_t per_chunk = (int64_t)g.tiles_j * g.tiles_k;
    const int64_t it0 = g.n_items * blockIdx.x / gridDim.x;
    const int64_t it1 = g.n_items * (blockIdx.x + 1) / gridDim.x;
    // this thread computes staged word (ty+1, tx+1): cur row word cw, row above cw-LTW
    const int cw = (ty + 1) * LTW + tx + 1;

    for (int64_t item = it0; item < it1; ++item) {
        const int64_t ch = item / per_chunk;
        const int rem = (int)(item - ch * per_chunk);
        const int j0 = (rem / g.tiles_k) * LCJ;
        const int k0 = (rem % g.tiles_k) * (2 * LCW);
        const int64_t ia = g.v0 + ch * g.chunk;
        const int64_t ib = min(ia + (int64_t)g.chunk, g.v1);

        // staged word (ty, tx) = cells (row j0-1+ty, cols k0-2+2tx and +1)
        const int jj = j0 - 1 + ty, kk = k0 - 2 + 2 * tx;
        const bool row_ok = jj >= 0 && jj < Wi && kk >= 0;
        const bool okx = row_ok && kk < Di, oky = row_ok && kk + 1 < Di;
        // pointer to this word in plane ia-1 (bumped by one plane per step)
        const T* ptr = buf + ((ia - 1 - g.first) * plane_elems + (okx ? (int64_t)jj * Di + kk : 0));
        // planes are addressed relative to ia-1: t = 0 .. n+1; plane ia-1+t
        // exists iff t_lo <= t < t_hi (32-bit, uniform)
        const int n = (int)(ib - ia);
        const int t_lo = ia >= 1 ? 0 : (int)(1 - ia);
        const int t_hi = (int)min((int64_t)(n + 2), g.H - ia + 1);
        auto fetch = [&](int t, const T* at) {
            const bool pin = t >= t_lo && t < t_hi;
            return load_pair<DT, VEC>(at, pin && okx, pin && oky);
        };
        auto store = [&](int t, uint32_t* dstp, const P2& v) {
            const bool pin = t >= t_lo && t < t_hi;
            dstp[tid] = pack_pair<DT, QM, SH>(v, pin && okx, pin && oky, tt, q, g.M, sent4);
        };
        // raw ring without register moves: ra feeds even steps, rb odd steps
        P2 ra = fetch(0, ptr);
        store(0, pl, ra);
        ra = fetch(1, ptr + plane_elems);
        P2 rb = fetch(2, ptr + 2 * plane_elems);
        ptr += 3 * plane_elems;  // next fetch: t = 3
        __syncthreads();

        // loaded words carry this lane's copy offset (no carry: lanes < 2^16)
        uint32_t W_ = pl[cw] + cpy, U = pl[cw - LTW] + cpy;
        uint32_t pW = W_;
        uint32_t pm2k = vmin2(W_, shift_pair(pl[cw - 1] + cpy, W_));
        uint32_t pm2j = vmin2(W_, U);
        uint32_t pm4i = vmin2(pm2k, vmin2(U, shift_pair(pl[cw - LTW - 1] + cpy, U)));

        auto step = [&](const uint32_t* cur) {
            if (!computes) return;
            W_ = cur[cw] + cpy;
            U = cur[cw - LTW] + cpy;
            const uint32_t Wm = shift_pair(cur[cw - 1] + cpy, W_);
            const uint32_t Um = shift_pair(cur[cw - LTW - 1] + cpy, U);
            const uint32_t m2k = vmin2(W_, Wm);             // face normal k
            const uint32_t m2j = vmin2(W_, U);              // face normal j
            const uint32_t m4i = vmin2(m2k, vmin2(U, Um));  // edge along i
            inc2(h, 0, hs, W_);
            inc2(h, 1, hs, vmin2(W_, pW));     // face normal i
            inc2(h, 1, hs, m2j);
            inc2(h, 1, hs, m2k);
            inc2(h, 2, hs, m4i);
            inc2(h, 2, hs, vmin2(m2k, pm2k));  // edge along j
            inc2(h, 2, hs, vmin2(m2j, pm2j));  // edge along k
            inc2(h, 3, hs, vmin2(m4i, pm4i));  // vertex
            pW = W_;
            pm2k = m2k;
            pm2j = m2j;
            pm4i = m4i;
        };
        for (int s = 0; s < n; s += 2) {
            // step s: lattice row ia+s from plane t = s+1 (buffer 1)
            uint32_t* cur = pl + LNT;
            store(s + 1, cur, ra);
            if (s + 2 < n) ra = fetch(s + 3, ptr);
            ptr += plane_elems;
            __syncthreads();
            step(cur);
            if (s + 1 >= n) break;
            cur = pl;  // step s+1: plane t = s+2 (buffer 0)
            store(s + 2, cur, rb);
            if (s + 3 < n) rb = fetch(s + 4, ptr);
            ptr += plane_elems;
            __syncthreads();
            step(cur);
        }
        __syncthreads();
    }
    __syncthreads();
    flush_rows<CP>(reinterpret_cast<uint32_t*>(h), hist, 4, M2, hs / 4, false);
}

// ------------------------------------------------ per-cell signatures
// The cube and its faces are booked ONCE per cell: a face appears at the
// level of whichever of its two cells activates first, so under the
// reference's total order -- level, then (k, j, i) lexicographic, the slot
// order of contrib3d.py:47-49 -- every face is owned by exactly one cell, and
// cell c contributes (1 cube, f faces) at its own level, f = #face
// neighbours that activate after c.  One increment of signature row u = 6 - f
// at level(c) replaces the cube event and three face events; the flush folds
// the seven signature rows into C = sum_u sig_u and F = sum_u (6 - u) sig_u.
// Edges and vertices stay min-filter events.  Cells of plane i are signed one
// step late (their +i neighbour arrives with plane i+1), so every slab/chunk
// covering lattice rows [a, b) signs cell planes [a-1, b-1): disjoint and
// complete.

// --------------------------------- 3D, register-blocked and barrier-free
// The per-cell signature booking (5 shared atomics per lattice point)
// without staging: every WARP independently owns a strip of R lattice
// rows x 60 lattice columns and marches the planes.  Lane l holds the words
// (two k-adjacent cells) of column pair l for the R+2 cell rows j0-1 .. j0+R
// of the current plane in registers, so j-neighbours are registers and
// k-neighbours one shuffle away; lanes 0 and 31 carry the halo columns.
// Each lane loads and quantizes its own words (one 8-byte load per row per
// plane, two planes in flight), so there is no shared staging, no LDS/STS and
// no CTA barrier: the shared memory serves only the histograms.
template <int DT, int QM, bool VEC, int R>
__global__ void __launch_bounds__(256, 2) lattice3d_rb_kernel(const typename Elem<DT>::T* __restrict__ buf, LGeo g,
                                                           QuantDev q, unsigned long long* __restrict__ hist)
{
    using P2 = typename Pair<DT>::T;
    using T = typename Elem<DT>::T;
    constexpr int NR = R + 2;                              // cell rows held per plane
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int M2 = g.M + 2;
    const int hs = g.hs;
    char* h = reinterpret_cast<char*>(smem_raw);           // rows: sig u = 0..6, edges, vertices
    float* tt = reinterpret_cast<float*>(h + 9 * hs);
    for (int i = threadIdx.x; i < 9 * hs / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(h)[i] = 0;
    if (QM != FT_Q_IDENTITY && QM != FT_Q_POW2)
        for (int i = threadIdx.x; i < M2; i += blockDim.x) tt[i] = q.tt[i];
    __syncthreads();
    char* hsig = h;
    char* hE = h + 7 * hs;
    char* hV = h + 8 * hs;

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x / 32;
    const bool computes = lane >= 1 && lane <= 30;
    const int Wi = (int)g.W, Di = (int)g.D;
    const int64_t plane_elems = g.W * g.D;
    const uint32_t sent4 = (uint32_t)(g.M + 1) * 4u;
    const uint32_t hs_pk = (uint32_t)hs;
    const int64_t per_chunk = (int64_t)g.tiles_j * g.tiles_k;

    // A CTA item is 8 vertically adjacent warp strips (8R lattice rows) x 60
    // columns x a chunk of planes: the warps march the same planes in
    // step, so the halo rows a warp shares with its neighbours are L1 hits.
    // Items are strided over CTAs so that concurrently running CTAs hold
    // adjacent column tiles and their halo columns meet in L2.
    for (int64_t item = blockIdx.x; item < g.n_items; item += gridDim.x) {
        const int64_t ch = item / per_chunk;
        const int rem = (int)(item - ch * per_chunk);
        const int j0 = (rem / g.tiles_k) * (8 * R) + warp * R;
        const int k0 = (rem % g.tiles_k) * 60;
        const int64_t ia = g.v0 + ch * g.chunk;
        const int64_t ib = min(ia + (int64_t)g.chunk, g.v1);
        const int kk = k0 - 2 + 2 * lane;
        const bool okx = kk >= 0 && kk < Di, oky = kk >= 0 && kk + 1 < Di;
        uint32_t rowok = 0;  // bit r: cell row j0-1+r exists (warp-uniform)
#pragma unroll
        for (int r = 0; r < NR; ++r) rowok |= (j0 - 1 + r >= 0 && j0 - 1 + r < Wi) ? 1u << r : 0u;
        const int n = (int)(ib - ia);
        const int t_lo = (int)max((int64_t)-1, 1 - ia);
        const int t_hi = (int)min((int64_t)(n + 2), g.H - ia + 1);
        // word of row 0 in plane ia-2 (t = -1); rows are D elements apart
        const T* ptr = buf + ((ia - 2 - g.first) * plane_elems + (int64_t)(j0 - 1) * Di + (okx ? kk : 0));
        auto fetch = [&](int t, const T* at, P2 (&dst)[NR]) {
            const bool pin = t >= t_lo && t < t_hi;
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                const bool ok = pin && ((rowok >> r) & 1u);
                dst[r] = load_pair<DT, VEC>(at + r * Di, ok && okx, ok && oky);
            }
        };
        const uint32_t lanekeep = (okx ? 0x0000FFFFu : 0u) | (oky ? 0xFFFF0000u : 0u);
        auto quant = [&](int t, const P2 (&src)[NR], uint32_t (&V)[NR]) {
            const bool pin = t >= t_lo && t < t_hi;
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                const bool ok = pin && ((rowok >> r) & 1u);
                if constexpr (QM == FT_Q_POW2)
                    V[r] = pack_pair_pow2<DT>(src[r], ok ? lanekeep : 0u, q.scale, (uint32_t)g.M * 0x10001u,
                                              sent4 * 0x10001u);
                else
                    V[r] = pack_pair<DT, QM, 0>(src[r], ok && okx, ok && oky, tt, q, g.M, sent4);
            }
        };

        uint32_t V[NR], pV[NR], tmi[NR], pWm[NR], pWp[NR], pm2k[NR], pm2j[NR], pm4i[NR];
        P2 ra[NR], rb[NR];
        // prologue: planes ia-2 (t = -1) and ia-1 (t = 0)
        fetch(-1, ptr, ra);
        fetch(0, ptr + plane_elems, rb);
        quant(-1, ra, V);
        quant(0, rb, pV);
        // "-i neighbour activates first" terms of the cells signed next: [V(ia-2) <= V(ia-1)]
#pragma unroll
        for (int r = 0; r < NR; ++r) tmi[r] = (((pV[r] | 0x80008000u) - V[r]) >> 15) & 0x10001u;
        fetch(1, ptr + 2 * plane_elems, ra);
        fetch(2, ptr + 3 * plane_elems, rb);
        ptr += 4 * plane_elems;  // next fetch: t = 3
        {
            uint32_t Wm[NR];
#pragma unroll
            for (int r = 0; r < NR; ++r) Wm[r] = shift_pair(__shfl_up_sync(0xFFFFFFFFu, pV[r], 1), pV[r]);
#pragma unroll
            for (int r = 1; r <= R; ++r) {
                pWm[r] = Wm[r];
                pWp[r] = shift_pair(pV[r], __shfl_down_sync(0xFFFFFFFFu, pV[r], 1));
                pm2k[r] = vmin2(pV[r], Wm[r]);
                pm2j[r] = vmin2(pV[r], pV[r - 1]);
                pm4i[r] = vmin2(pm2k[r], vmin2(pV[r - 1], Wm[r - 1]));
            }
        }

        auto step = [&]() {
            uint32_t Wm[NR], ev[R + 1][5], tpj = 0;
#pragma unroll
            for (int r = 0; r < NR; ++r) Wm[r] = shift_pair(__shfl_up_sync(0xFFFFFFFFu, V[r], 1), V[r]);
#pragma unroll
            for (int r = 1; r <= R; ++r) {
                const uint32_t W_ = V[r], U = V[r - 1];
                const uint32_t Wp = shift_pair(W_, __shfl_down_sync(0xFFFFFFFFu, W_, 1));
                const uint32_t m2k = vmin2(W_, Wm[r]);             // face normal k
                const uint32_t m2j = vmin2(W_, U);                 // face normal j
                const uint32_t m4i = vmin2(m2k, vmin2(U, Wm[r - 1]));  // edge along i
                ev[r][0] = m4i;
                ev[r][1] = vmin2(m2k, pm2k[r]);  // edge along j
                ev[r][2] = vmin2(m2j, pm2j[r]);  // edge along k
                ev[r][3] = vmin2(m4i, pm4i[r]);  // vertex
                // signature of the plane-(i-1) cells of row r (per-cell signatures, above).
                // Each term is bit 15 / 31 of c' - n + k: "n activates before c".
                // The -i term is the complement of the previous step's +i term and
                // the -j term (rows >= 2) the complement of row r-1's +j term.
                const uint32_t cb = pV[r] | 0x80008000u;
                const uint32_t t1 = r == 1 ? ((cb - pV[0]) >> 15) & 0x10001u : 0x10001u - tpj;  // -j
                const uint32_t t2 = ((cb - pWm[r]) >> 15) & 0x10001u;                             // -k
                const uint32_t t3 = ((cb - W_ - 0x10001u) >> 15) & 0x10001u;                      // +i
                const uint32_t t4 = ((cb - pV[r + 1] - 0x10001u) >> 15) & 0x10001u;               // +j
                const uint32_t t5 = ((cb - pWp[r] - 0x10001u) >> 15) & 0x10001u;                  // +k
                const uint32_t u = tmi[r] + t1 + t2 + t3 + t4 + t5;
                ev[r][4] = u * hs_pk + pV[r];
                tmi[r] = 0x10001u - t3;
                tpj = t4;
                pWm[r] = Wm[r];
                pWp[r] = Wp;
                pm2k[r] = m2k;
                pm2j[r] = m2j;
                pm4i[r] = m4i;
            }
#pragma unroll
            for (int r = 0; r < NR; ++r) pV[r] = V[r];
            if (computes) {  // one divergent region per step (lanes 0 / 31 carry halos)
#pragma unroll
                for (int r = 1; r <= R; ++r) {
                    inc2(hE, 0, hs, ev[r][0]);
                    inc2(hE, 0, hs, ev[r][1]);
                    inc2(hE, 0, hs, ev[r][2]);
                    inc2(hV, 0, hs, ev[r][3]);
                    inc2(hsig, 0, hs, ev[r][4]);
                }
            }
        };
        for (int s = 0; s < n; s += 2) {
            quant(s + 1, ra, V);  // plane t = s+1
            if (s + 2 < n) fetch(s + 3, ptr, ra);
            ptr += plane_elems;
            step();
            if (s + 1 >= n) break;
            quant(s + 2, rb, V);
            if (s + 3 < n) fetch(s + 4, ptr, rb);
            ptr += plane_elems;
            step();
        }
    }
    __syncthreads();
    const uint32_t* hw = reinterpret_cast<const uint32_t*>(h);
    const int rw = hs / 4;
    for (int l = threadIdx.x; l < M2; l += blockDim.x) {
        uint32_t c = 0, f = 0;
#pragma unroll
        for (int u = 0; u < 7; ++u) {
            const uint32_t v = hw[u * rw + l];
            c += v;
            f += (6 - u) * v;
        }
        const uint32_t e = hw[7 * rw + l], x = hw[8 * rw + l];
        if (c) atomicAdd(&hist[l], (unsigned long long)c);
        if (f) atomicAdd(&hist[M2 + l], (unsigned long long)f);
        if (e) atomicAdd(&hist[2 * M2 + l], (unsigned long long)e);
        if (x) atomicAdd(&hist[3 * M2 + l], (unsigned long long)x);
    }
}

// ------------------------------------------------------------------- 2D
// Lattice point p = (i, j) owns the cell (i, j), the edge to (i, j+1) (cells
// (i-1, j), (i, j)), the edge to (i+1, j) (cells (i, j-1), (i, j)) and its
// low-corner vertex (cells (i-1..i, j-1..j)).  Rows: cells, edge mins, vertex
// mins, vertex maxes (the last only for EC_4C; E_max = 4C - E is implied).
// A 256-thread CTA stages one row segment of 256 words per step (one per
// thread) and 255 threads compute 510 lattice columns.
constexpr int L2W = 256;
constexpr int L2C = L2W - 1;

template <int DT, int QM, bool MAXES, bool VEC, int CP>
__global__ void __launch_bounds__(L2W) lattice2d_kernel(const typename Elem<DT>::T* __restrict__ buf, LGeo g,
                                                         QuantDev q, unsigned long long* __restrict__ hist)
{
    using P2 = typename Pair<DT>::T;
    using T = typename Elem<DT>::T;
    constexpr int SH = Priv<CP>::SH;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int M2 = g.M + 2;
    constexpr int NR = 4;
    const int hs = g.hs;
    char* h = reinterpret_cast<char*>(smem_raw);
    float* tt = reinterpret_cast<float*>(h + NR * hs);
    uint32_t* rows = reinterpret_cast<uint32_t*>(tt + M2);  // [2][L2W]
    for (int i = threadIdx.x; i < hs; i += L2W) reinterpret_cast<uint32_t*>(h)[i] = 0;
    if (QM != FT_Q_IDENTITY)
        for (int i = threadIdx.x; i < M2; i += L2W) tt[i] = q.tt[i];
    __syncthreads();

    const int tid = threadIdx.x;
    const bool computes = tid < L2C;
    const uint32_t sent4 = ((uint32_t)(g.M + 1) * 4u) << SH;
    const uint32_t cpy = (uint32_t)(tid % CP) * 4u * 0x10001u;
    const int Wi = (int)g.W;
    const int64_t it0 = g.n_items * blockIdx.x / gridDim.x;
    const int64_t it1 = g.n_items * (blockIdx.x + 1) / gridDim.x;
    int64_t cur_img = it0 < it1 ? it0 / g.items_per_image : 0;

    for (int64_t item = it0; item < it1; ++item) {
        const int64_t b = item / g.items_per_image;
        if (b != cur_img) {  // histograms belong to one image: flush on change
            __syncthreads();
            flush_rows<CP>(reinterpret_cast<uint32_t*>(h), hist + cur_img * NR * M2, NR, M2, hs / 4, true);
            __syncthreads();
            cur_img = b;
        }
        const int64_t rem = item - b * g.items_per_image;
        const int64_t ch = rem / g.tiles_k;
        const int j0 = (int)(rem % g.tiles_k) * (2 * L2C);
        const int64_t ia = g.v0 + ch * g.chunk;
        const int64_t ib = min(ia + (int64_t)g.chunk, g.v1);
        // staged word tid = cells (j0-2+2tid, +1); thread tid computes word tid+1
        const int kk = j0 - 2 + 2 * tid;
        const bool okx = kk >= 0 && kk < Wi, oky = kk >= 0 && kk + 1 < Wi;
        const T* ptr = buf + b * g.bstride + ((ia - 1 - g.first) * g.W + (okx ? kk : 0));
        // rows relative to ia-1: t = 0 .. n+1 (see the 3D kernel)
        const int n = (int)(ib - ia);
        const int t_lo = ia >= 1 ? 0 : (int)(1 - ia);
        const int t_hi = (int)min((int64_t)(n + 2), g.H - ia + 1);
        auto fetch = [&](int t, const T* at) {
            const bool rin = t >= t_lo && t < t_hi;
            return load_pair<DT, VEC>(at, rin && okx, rin && oky);
        };
        auto store = [&](int t, uint32_t* dst, const P2& v) {
            const bool rin = t >= t_lo && t < t_hi;
            dst[tid] = pack_pair<DT, QM, SH>(v, rin && okx, rin && oky, tt, q, g.M, sent4);
        };
        P2 ra = fetch(0, ptr);
        store(0, rows, ra);
        ra = fetch(1, ptr + g.W);
        P2 rb = fetch(2, ptr + 2 * g.W);
        ptr += 3 * g.W;
        __syncthreads();
        uint32_t pW = rows[tid + 1] + cpy;
        uint32_t pWm = shift_pair(rows[tid] + cpy, pW);
        auto step = [&](const uint32_t* cur) {
            if (!computes) return;
            const uint32_t W_ = cur[tid + 1] + cpy;
            const uint32_t Wm = shift_pair(cur[tid] + cpy, W_);
            const uint32_t ev = vmin2(W_, Wm);  // edge (i,j)-(i+1,j): cells (i,j-1), (i,j)
            inc2(h, 0, hs, W_);
            inc2(h, 1, hs, vmin2(W_, pW));  // edge (i,j)-(i,j+1): cells (i-1,j), (i,j)
            inc2(h, 1, hs, ev);
            inc2(h, 2, hs, vmin2(ev, vmin2(pW, pWm)));
            if constexpr (MAXES) inc2(h, 3, hs, vmax2(vmax2(W_, Wm), vmax2(pW, pWm)));
            pW = W_;
            pWm = Wm;
        };
        for (int s = 0; s < n; s += 2) {
            uint32_t* cur = rows + L2W;
            store(s + 1, cur, ra);
            if (s + 2 < n) ra = fetch(s + 3, ptr);
            ptr += g.W;
            __syncthreads();
            step(cur);
            if (s + 1 >= n) break;
            cur = rows;
            store(s + 2, cur, rb);
            if (s + 3 < n) rb = fetch(s + 4, ptr);
            ptr += g.W;
            __syncthreads();
            step(cur);
        }
        __syncthreads();
    }
    __syncthreads();
    if (it0 < it1) flush_rows<CP>(reinterpret_cast<uint32_t*>(h), hist + cur_img * NR * M2, NR, M2, hs / 4, false);
}

// ------------------------------------------- 2D, register march + signatures
// Same rows as lattice2d_kernel.  A 64-thread CTA (two warps, one shared
// histogram set) owns 2 x 60 lattice columns of one image and a chunk of
// rows; every lane marches its two k-adjacent cells down the rows with the
// previous rows in registers and the j-neighbours one shuffle away (lanes 0
// and 31 carry the halo columns).  Cells and edges are booked once per cell
// (signature u = #edge neighbours that activate first under the reference's
// row-major order, contrib2d.py:39-40: E = sum (4 - u) sig_u), vertices by
// their min (and max for EC_4C): 2-3 shared atomics per lattice point.
template <int DT, int QM, bool MAXES, bool VEC>
__global__ void __launch_bounds__(64) lattice2d_rb_kernel(const typename Elem<DT>::T* __restrict__ buf, LGeo g,
                                                          QuantDev q, unsigned long long* __restrict__ hist)
{
    using P2 = typename Pair<DT>::T;
    using T = typename Elem<DT>::T;
    constexpr int NR = 4;      // output rows: cells, edges, vertices, vertex maxes
    constexpr int PF = 4;      // rows in flight per lane
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int M2 = g.M + 2;
    const int hs = g.hs;
    char* h = reinterpret_cast<char*>(smem_raw);  // rows: sig u = 0..4, vertices, vertex maxes
    float* tt = reinterpret_cast<float*>(h + 7 * hs);
    for (int i = threadIdx.x; i < 7 * hs / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(h)[i] = 0;
    if (QM != FT_Q_IDENTITY && QM != FT_Q_POW2)
        for (int i = threadIdx.x; i < M2; i += blockDim.x) tt[i] = q.tt[i];
    __syncthreads();
    char* hsig = h;
    char* hV = h + 5 * hs;
    char* hX = h + 6 * hs;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool computes = lane >= 1 && lane <= 30;
    const int Wi = (int)g.W;
    const uint32_t sent4 = (uint32_t)(g.M + 1) * 4u;
    const uint32_t hs_pk = (uint32_t)hs;
    const uint32_t halo4 = computes ? 0u : sent4 * 0x10001u;

    auto flush = [&](int64_t img, bool zero) {
        __syncthreads();
        uint32_t* hw = reinterpret_cast<uint32_t*>(h);
        const int rw = hs / 4;
        unsigned long long* out = hist + img * NR * M2;
        for (int l = threadIdx.x; l < M2; l += blockDim.x) {
            uint32_t c = 0, e = 0;
#pragma unroll
            for (int u = 0; u < 5; ++u) {
                const uint32_t v = hw[u * rw + l];
                c += v;
                e += (4 - u) * v;
                if (zero) hw[u * rw + l] = 0;
            }
            const uint32_t x = hw[5 * rw + l], y = hw[6 * rw + l];
            if (zero) hw[5 * rw + l] = hw[6 * rw + l] = 0;
            if (c) atomicAdd(&out[l], (unsigned long long)c);
            if (e) atomicAdd(&out[M2 + l], (unsigned long long)e);
            if (x) atomicAdd(&out[2 * M2 + l], (unsigned long long)x);
            if (y) atomicAdd(&out[3 * M2 + l], (unsigned long long)y);
        }
        __syncthreads();
    };

    int64_t cur_img = -1;
    for (int64_t item = blockIdx.x; item < g.n_items; item += gridDim.x) {
        const int64_t b = item / g.items_per_image;
        if (b != cur_img) {
            if (cur_img >= 0) flush(cur_img, true);
            cur_img = b;
        }
        const int64_t rem = item - b * g.items_per_image;
        const int64_t ch = rem / g.tiles_k;
        const int k0 = (int)(rem % g.tiles_k) * 120 + warp * 60;
        const int64_t ia = g.v0 + ch * g.chunk;
        const int64_t ib = min(ia + (int64_t)g.chunk, g.v1);
        const int kk = k0 - 2 + 2 * lane;
        const bool okx = kk >= 0 && kk < Wi, oky = kk >= 0 && kk + 1 < Wi;
        const uint32_t lanekeep = (okx ? 0x0000FFFFu : 0u) | (oky ? 0xFFFF0000u : 0u);
        const int n = (int)(ib - ia);
        const int t_lo = (int)max((int64_t)-1, 1 - ia);
        const int t_hi = (int)min((int64_t)(n + 2), g.H - ia + 1);
        const T* ptr = buf + b * g.bstride + ((ia - 2 - g.first) * g.W + (okx ? kk : 0));
        auto fetch = [&](int t) {
            const bool pin = t >= t_lo && t < t_hi;
            return load_pair<DT, VEC>(ptr + (int64_t)(t + 1) * g.W, pin && okx, pin && oky);
        };
        auto quant = [&](int t, const P2& v, bool inside) -> uint32_t {
            const bool pin = inside || (t >= t_lo && t < t_hi);
            if constexpr (QM == FT_Q_POW2)
                return pack_pair_pow2<DT>(v, pin ? lanekeep : 0u, q.scale, (uint32_t)g.M * 0x10001u,
                                          sent4 * 0x10001u);
            else
                return pack_pair<DT, QM, 0>(v, pin && okx, pin && oky, tt, q, g.M, sent4);
        };
        // rows relative to ia-1: t = -1 .. n (row ia-1+t)
        const uint32_t r_m1 = quant(-1, fetch(-1), false);
        uint32_t pW = quant(0, fetch(0), false);  // row ia-1
        P2 raw[PF];
#pragma unroll
        for (int p = 0; p < PF; ++p) raw[p] = fetch(1 + p);
        uint32_t pWm = shift_pair(__shfl_up_sync(0xFFFFFFFFu, pW, 1), pW);
        uint32_t pWp = shift_pair(pW, __shfl_down_sync(0xFFFFFFFFu, pW, 1));
        uint32_t tmi = (((pW | 0x80008000u) - r_m1) >> 15) & 0x10001u;  // [row ia-2 <= row ia-1]

        // One lattice row.  The halo lanes 0 and 31 book into the sentinel
        // bin M+1 (never read: curves stop at level M) instead of branching.
        auto step = [&](uint32_t W_) {
            const uint32_t Wm = shift_pair(__shfl_up_sync(0xFFFFFFFFu, W_, 1), W_);
            const uint32_t Wp = shift_pair(W_, __shfl_down_sync(0xFFFFFFFFu, W_, 1));
            const uint32_t ev = vmin2(W_, Wm);              // edge (i,j)-(i+1,j)
            const uint32_t vx = vmin2(ev, vmin2(pW, pWm));  // vertex
            // signature of the row-(i-1) cells pW
            const uint32_t cb = pW | 0x80008000u;
            const uint32_t t_mj = ((cb - pWm) >> 15) & 0x10001u;             // -j
            const uint32_t t_pj = ((cb - pWp - 0x10001u) >> 15) & 0x10001u;  // +j
            const uint32_t t_pi = ((cb - W_ - 0x10001u) >> 15) & 0x10001u;   // +i
            const uint32_t u = tmi + t_mj + t_pj + t_pi;
            inc2(hsig, 0, hs, u * hs_pk + vmax2(pW, halo4));
            inc2(hV, 0, hs, vmax2(vx, halo4));
            if constexpr (MAXES) inc2(hX, 0, hs, vmax2(vmax2(W_, Wm), vmax2(vmax2(pW, pWm), halo4)));
            tmi = 0x10001u - t_pi;
            pW = W_;
            pWm = Wm;
            pWp = Wp;
        };
        // steady state: every row fetched and quantized is inside the image
        const int S = min(n - PF, t_hi - 1 - PF);
        int s0 = 0;
        for (; s0 + PF <= S; s0 += PF) {
#pragma unroll
            for (int p = 0; p < PF; ++p) {
                const int s = s0 + p;
                const uint32_t W_ = quant(s + 1, raw[p], true);
                raw[p] = load_pair<DT, VEC>(ptr + (int64_t)(s + 2 + PF) * g.W, okx, oky);
                step(W_);
            }
        }
        for (; s0 < n; s0 += PF) {
#pragma unroll
            for (int p = 0; p < PF; ++p) {
                const int s = s0 + p;
                if (s >= n) break;
                const uint32_t W_ = quant(s + 1, raw[p], false);
                if (s + PF < n) raw[p] = fetch(s + 1 + PF);
                step(W_);
            }
        }
    }
    if (cur_img >= 0) flush(cur_img, false);
}


template <int DT, int QM>
static int launch_l3(const ft_window* win, int64_t H, int64_t W, int64_t D, int64_t v0, int64_t v1,
                     const ft_quant* qa, int32_t M, uint64_t* hist, cudaStream_t st)
{
    using T = typename Elem<DT>::T;
    LGeo g{};
    g.H = H; g.W = W; g.D = D; g.v0 = v0; g.v1 = v1; g.first = win->first; g.M = M;
    const bool vec3 = D % 2 == 0 && reinterpret_cast<uintptr_t>(win->data) % 8 == 0;
    if (6 * (((M + 2) * 4 + 15) / 16 * 16) + (M + 1) * 4 < 0xFFFF) {
        // R = 6 rows per warp strip: 127 registers, 2 CTAs/SM; measured at
        // 2048^3: R=4 451, R=6 479, R=8 384 (spills), R=4 forced to 3 CTAs 440 Gvox/s
        constexpr int R = 6, NTH = 256;
        g.hs = ((M + 2) * 4 + 15) / 16 * 16;
        const size_t smem = (size_t)9 * g.hs + (size_t)(M + 2) * 4;
        auto kern = vec3 ? lattice3d_rb_kernel<DT, QM, true, R> : lattice3d_rb_kernel<DT, QM, false, R>;
        FT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        FT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NTH, smem));
        if (per_sm < 1) return FT_ERR_ARG;
        g.tiles_j = (int)cdiv(W + 1, (NTH / 32) * R);  // CTA items: 8 warp strips
        g.tiles_k = (int)cdiv(D + 1, 60);
        const int64_t grid_cap = (int64_t)nsm_l() * per_sm;
        plan_items(g, (int64_t)g.tiles_j * g.tiles_k, 1, grid_cap, 64);
        const int grid = (int)std::min<int64_t>(grid_cap, g.n_items);
        kern<<<grid, NTH, smem, st>>>(static_cast<const T*>(win->data), g, qdev(qa),
                                      reinterpret_cast<unsigned long long*>(hist));
        FT_CUDA_TRY(cudaGetLastError());
        return FT_OK;
    }
    // larger level counts: the staged kernel (one histogram copy; measured,
    // profiles/r01/lattice_notes.md: privatised copies do not lower the
    // conflict degree on smooth fields)
    g.hs = row_stride(M, 1);
    const size_t smem = (size_t)4 * g.hs + (size_t)(M + 2) * 4 + 2 * LNT * 4;
    const bool vec = D % 2 == 0 && reinterpret_cast<uintptr_t>(win->data) % 8 == 0;
    auto kern = vec ? lattice3d_kernel<DT, QM, true, 1> : lattice3d_kernel<DT, QM, false, 1>;
    FT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    FT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, LNT, smem));
    if (per_sm < 1) return FT_ERR_ARG;
    // lattice points j in [0, W], k in [0, D] (the high boundary included)
    g.tiles_j = (int)cdiv(W + 1, LCJ);
    g.tiles_k = (int)cdiv(D + 1, 2 * LCW);
    const int64_t grid_cap = (int64_t)nsm_l() * per_sm;
    plan_items(g, (int64_t)g.tiles_j * g.tiles_k, 1, grid_cap, 32);
    const int grid = (int)std::min<int64_t>(grid_cap, g.n_items);
    kern<<<grid, LNT, smem, st>>>(static_cast<const T*>(win->data), g, qdev(qa),
                                  reinterpret_cast<unsigned long long*>(hist));
    FT_CUDA_TRY(cudaGetLastError());
    return FT_OK;
}

template <int DT, int QM>
static int launch_l2(const ft_window* win, int64_t H, int64_t W, int64_t v0, int64_t v1, const ft_quant* qa,
                     int32_t M, int maxes, uint64_t* hist, cudaStream_t st)
{
    using T = typename Elem<DT>::T;
    LGeo g{};
    g.H = H; g.W = W; g.D = 1; g.v0 = v0; g.v1 = v1; g.first = win->first; g.M = M;
    g.bstride = win->batch_stride;
    g.hs = row_stride(M, 1);
    const int64_t batch = std::max<int64_t>(win->batch, 1);
    const size_t smem = (size_t)4 * g.hs + (size_t)(M + 2) * 4 + 2 * L2W * 4;
    const bool vec = W % 2 == 0 && (batch <= 1 || win->batch_stride % 2 == 0) &&
                     reinterpret_cast<uintptr_t>(win->data) % 8 == 0;
    const int hs_rb = ((M + 2) * 4 + 15) / 16 * 16;
    if (4 * hs_rb + (M + 1) * 4 < 0xFFFF) {
        g.hs = hs_rb;
        const size_t smem_rb = (size_t)7 * hs_rb + (size_t)(M + 2) * 4;
        using K = void (*)(const T*, LGeo, QuantDev, unsigned long long*);
        K kern = maxes ? (vec ? lattice2d_rb_kernel<DT, QM, true, true> : lattice2d_rb_kernel<DT, QM, true, false>)
                       : (vec ? lattice2d_rb_kernel<DT, QM, false, true> : lattice2d_rb_kernel<DT, QM, false, false>);
        FT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_rb));
        int per_sm = 0;
        FT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 64, smem_rb));
        if (per_sm < 1) return FT_ERR_ARG;
        g.tiles_k = (int)cdiv(W + 1, 120);
        const int64_t grid_cap = (int64_t)nsm_l() * per_sm;
        // about one item per CTA (equal work), marches of >= 64 rows
        const int64_t rows = v1 - v0;
        int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>(cdiv(grid_cap, g.tiles_k * batch), rows / 64));
        g.chunk = (int)cdiv(rows, nchunks);
        nchunks = cdiv(rows, g.chunk);
        g.items_per_image = g.tiles_k * nchunks;
        g.n_items = g.items_per_image * batch;
        const int grid = (int)std::min<int64_t>(grid_cap, g.n_items);
        kern<<<grid, 64, smem_rb, st>>>(static_cast<const T*>(win->data), g, qdev(qa),
                                        reinterpret_cast<unsigned long long*>(hist));
        FT_CUDA_TRY(cudaGetLastError());
        return FT_OK;
    }
    // larger level counts: the staged kernel (one histogram copy)
    using K = void (*)(const T*, LGeo, QuantDev, unsigned long long*);
    K kern = maxes ? (vec ? lattice2d_kernel<DT, QM, true, true, 1> : lattice2d_kernel<DT, QM, true, false, 1>)
                   : (vec ? lattice2d_kernel<DT, QM, false, true, 1> : lattice2d_kernel<DT, QM, false, false, 1>);
    FT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    FT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, L2W, smem));
    if (per_sm < 1) return FT_ERR_ARG;
    g.tiles_k = (int)cdiv(W + 1, 2 * L2C);
    const int64_t grid_cap = (int64_t)nsm_l() * per_sm;
    plan_items(g, g.tiles_k, batch, grid_cap, 64);
    const int grid = (int)std::min<int64_t>(grid_cap, g.n_items);
    kern<<<grid, L2W, smem, st>>>(static_cast<const T*>(win->data), g, qdev(qa),
                                  reinterpret_cast<unsigned long long*>(hist));
    FT_CUDA_TRY(cudaGetLastError());
    return FT_OK;
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
        if (qm == FT_Q_TABLE || qm == FT_Q_POW2) return LAUNCH<FT_U8, FT_Q_TABLE>(__VA_ARGS__); \
        return LAUNCH<FT_U8, FT_Q_TABLE_ROBUST>(__VA_ARGS__);                              \
    case FT_U16:                                                                           \
        if (qm == FT_Q_IDENTITY) return LAUNCH<FT_U16, FT_Q_IDENTITY>(__VA_ARGS__);        \
        if (qm == FT_Q_POW2) return LAUNCH<FT_U16, FT_Q_POW2>(__VA_ARGS__);                \
        if (qm == FT_Q_TABLE) return LAUNCH<FT_U16, FT_Q_TABLE>(__VA_ARGS__);              \
        return LAUNCH<FT_U16, FT_Q_TABLE_ROBUST>(__VA_ARGS__);                             \
    case FT_F32:                                                                           \
        if (qm == FT_Q_IDENTITY) return FT_ERR_ARG;                                        \
        if (qm == FT_Q_POW2) return LAUNCH<FT_F32, FT_Q_POW2>(__VA_ARGS__);                \
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
    if (!window_ok(win, H, v0, v1, 2)) return FT_ERR_ARG;
    const int qm = effective_qmode(q, true);
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
    const int qm = effective_qmode(q, true);
    if (qm != FT_Q_IDENTITY && !q->thresholds) return FT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    FT_LDISPATCH(launch_l2, win, H, W, v0, v1, q, M, maxes, hist, st)
}
