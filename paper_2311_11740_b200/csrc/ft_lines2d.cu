// ft_lines2d.cu -- fused EC (8C) / perimeter / area histograms of 2D fields
// and batches of them by line decomposition: the 2D counterpart of
// ft_lines.cu.
//
// The reference builds the 2D curves from per-vertex transition counts
// (contrib2d.py:161-232) folded with the weight tables (descriptors.py:
// 169-178).  ft_lattice.cu restates them as element counts by level
// (EC_8C = V - E + C, perimeter = 2E - 4C, area = C) with one dense vertex
// event per lattice point.  Here the vertices come from sparse events:
//
// * Slicing the closed pixel complex along the lattice lines between columns
//   (the closed line x = j, j = 0..W, and the open strips between them,
//   chi_c(open strip) = -chi of its column) gives
//       chi_2D = sum over i-lines of chi1(B) - chi1(A),
//   A = cell levels of a column, B = min over columns (j-1, j), both on the
//   lattice columns j in [0, W] (sentinel cells outside).  A line of unit
//   intervals has chi1 = sum of +1 (local minimum along i) / -1 (local
//   maximum), ties lower-i-first: ~10 % of the cells of a smooth field.
// * Cells and edges are booked once per cell by signature: row u + 5 (s + 1),
//   u = #edge neighbours activating first under the (level, index) order (so
//   E = sum (4 - u)), s = the cell's own A-line event.
//
// Per 64 cells: 2 dense ATOMS (signature) + 2 sparse (B events), against 4
// dense for lattice2d_rb_kernel.  Output rows per image (uint64 [4][M+2],
// accumulated, the lattice2d layout): C, E, V = EC + E - C; row 3 (vertex
// maxes, EC_4C) is left to ft_lattice2d.
#include "ft_lines.cuh"

namespace ft {

constexpr int L2L_NTH = 512;  // 16 warps, each a 62-column strip
// rows per (row block, column tile) piece (measured 64 / 96 / 128 / 256:
// profiles/r02/s3/ab_lines2d_rb.log)
#ifndef L2B_PF
#define L2B_PF 6
#endif
#ifndef L2B_MINB
#define L2B_MINB 2
#endif
constexpr int L2L_RB = 96;
constexpr int L2L_SIG = 15;        // signature rows u + 5 (s + 1)

// One warp strip: lattice columns k0 .. k0+61 of one image, lattice rows
// [ia, ib).  Lane l holds cells (kk, kk+1), kk = k0-1+2l; lane 0 computes its
// high half, lane 31 its low half (as in ft_lines.cu).  EDGE: columns outside
// the image (clamped pair loads, masked halves).
// PF: rows in flight per lane (even: the ping-pong march state).  WS > 0: the
// row stride W as a compile-time constant, so the PF row loads of a step are
// immediate offsets from one pointer (no 64-bit address math per row).
template <int DT, int QM, bool VEC, bool EDGE, int PF, int WS>
__device__ __forceinline__ void lines2d_item(const typename Elem<DT>::T* __restrict__ img, const LGeo& g,
                                             const QuantDev& q, const float* __restrict__ tt, uint32_t topd_u,
                                             uint32_t topp_u, int64_t ia, int64_t ib, int k0, int lane)
{
    using P2 = typename Pair<DT>::T;
    using T = typename Elem<DT>::T;
    constexpr uint32_t FULL = 0xFFFFFFFFu;
    const int Wi = WS > 0 ? WS : (int)g.W;
    const int64_t Ws = WS > 0 ? (int64_t)WS : g.W;  // row stride (elements)
    const uint32_t sent4 = (uint32_t)(g.M + 1) * 4u;
    constexpr uint32_t sbw = LINES_REL0;  // packed words: (level + 1) * 4 per half
    const uint32_t S2 = sent4 * 0x10001u + sbw;
    const uint32_t sent_lv2 = (uint32_t)(g.M + 1) * 0x10001u;
    const uint32_t hk = (uint32_t)g.hk;
    const float Mf = (float)g.M;
    const int kk = k0 - 1 + 2 * lane;
    const uint32_t lmask = __shfl_sync(FULL, lane == 0 ? 0xFFFF0000u : lane == 31 ? 0x0000FFFFu : FULL, lane);
    const uint32_t lsel = __shfl_sync(FULL, lane_sel(lane), lane);  // dense events: halo halves -> the dummy word
    // the region tops as per-lane registers (as uniform values ptxas puts a move in front of every IDP)
    const uint32_t topd = __shfl_sync(FULL, topd_u, lane), topp = __shfl_sync(FULL, topp_u, lane);
    const int n = (int)(ib - ia);
    // rows t = -1 .. n (row ia-1+t) exist iff t_lo <= t < t_hi; rows t < tf
    // are fetched (a window holds rows ia-2 .. ib-1)
    const int t_lo = (int)max((int64_t)-1, 1 - ia);
    const int t_hi = (int)min((int64_t)(n + 2), g.H - ia + 1);
    const int tf = min(n + 1, t_hi);
    const bool okx = kk >= 0 && kk < Wi, oky = kk + 1 >= 0 && kk + 1 < Wi;
    const uint32_t lanekeep = (okx ? 0x0000FFFFu : 0u) | (oky ? 0xFFFF0000u : 0u);
    const int kc = !EDGE ? kk : VEC ? min(max(kk, 0), Wi - 2) : min(max(kk, 0), Wi - 1);
    const T* ptr = img + ((ia - 2 - g.first) * Ws + kc);  // row ia-2 (t = -1)

    auto fetch = [&](int t, const T* at, P2& dst) {
        if (t >= t_lo && t < tf) dst = load_pair<DT, VEC>(at, true, EDGE ? kk + 1 < Wi : true);
    };
    auto quant_in = [&](const P2& src) -> uint32_t {
        uint32_t v;
        if constexpr (QM == FT_Q_POW2)
            v = pack_pow2_sat<DT>(src, q.inv, Mf, g.four, sbw);
        else if constexpr (QM == FT_Q_UMAGIC)
            v = pack_pair_umagic<DT>(src, q, g.four, sbw);  // u8 / u16 integer ranges: exact integer decoding
        else if constexpr (QM == FT_Q_IDENTITY && (DT == FT_U8 || DT == FT_U16))
            v = pack_pair_ident<DT>(src, sent_lv2, g.four, sbw);
        else
            v = pack_pair<DT, QM, 0>(src, true, true, tt, q, g.M, sent4) + sbw;
        return EDGE ? sel_mask(lanekeep, v, S2) : v;
    };
    auto quant = [&](int t, const P2& src) -> uint32_t { return t >= t_lo && t < t_hi ? quant_in(src) : S2; };

    struct St {
        uint32_t pV, pt3, pWm, pC, eC;  // pt3: the +i term t3 of the row before (tmi = 255 - pt3)
    };
    St sa, sb;
    P2 raw[PF];  // rows in flight: raw[p] holds row t = p+1 (mod PF)
    {
        P2 r0, r1;
        fetch(-1, ptr, r0);
        fetch(0, ptr + Ws, r1);
        const uint32_t V0 = quant(-1, r0);
        sa.pV = quant(0, r1);
        const uint32_t Wm0 = shift_pair(__shfl_up_sync(FULL, V0, 1), V0);
        sa.pWm = shift_pair(__shfl_up_sync(FULL, sa.pV, 1), sa.pV);
        const uint32_t C0 = vmin2(V0, Wm0);
        sa.pC = vmin2(sa.pV, sa.pWm);
        sa.pt3 = hff(cmp2(V0, sa.pV)) ^ FF2;  // the -i neighbour (row ia-2) does NOT activate first
        sa.eC = cmp2(C0, sa.pC);
    }
#pragma unroll
    for (int p = 0; p < PF; ++p) fetch(p + 1, ptr + (p + 2) * Ws, raw[p]);
    ptr += (PF + 2) * Ws;  // row t = PF+1

    // row t arrives in V; every event of the row before it (state o) is booked
    auto step = [&](uint32_t V, const St& o, St& x) {
        const uint32_t Wm = shift_pair(__shfl_up_sync(FULL, V, 1), V);
        const uint32_t Cn = vmin2(V, Wm);
        const uint32_t cb = o.pV | 0x80008000u;
        const uint32_t t2 = hff(cb - o.pWm);            // -j neighbour first
        const uint32_t t3 = hff(cb - V - 0x10001u);     // +i neighbour first
        // +j: complement of the right neighbour's -j term
        const uint32_t sh5 = shift_pair(t2, __shfl_down_sync(FULL, t2, 1));
        // row u + 5 (s + 1) = t2 + t5 + 10 - 4 (tmi + t3) in units of 255, with
        // t5 = 255 - sh5 and tmi = 255 - pt3: packed adds, constants folded;
        // every half ends in [0, 14 * 255] (intermediate borrows cancel)
        const uint32_t row = t2 - sh5 + 4u * (o.pt3 - t3) + 7u * FF2;
        sinc2(row * hk + o.pV, lsel, topd);
        // B line (min over columns j-1, j): +1 at a local min (plus row), -1
        // at a local max (minus row)
        const uint32_t nC = cmp2(o.pC, Cn);
        sinc2(o.pC | (~nC & 0x80008000u), ev_sel((o.eC ^ nC) & lmask), topp);
        x.pt3 = t3;
        x.pWm = Wm;
        x.pC = Cn;
        x.eC = nC;
        x.pV = V;
    };

    // steps s < nm see an existing row t = s+1; only the last step of the
    // image's last segment (row H) can follow, with a sentinel row
    const int nm = min(n, t_hi - 1);
    int s = 0;
    // steady state: 4 steps per iteration, every refill (rows s+5 .. s+8)
    // inside the segment -- no guards
    for (; s + PF <= nm && s + 2 * PF < tf; s += PF) {
#pragma unroll
        for (int p = 0; p < PF; ++p) {
            const uint32_t V = quant_in(raw[p]);
            raw[p] = load_pair<DT, VEC>(ptr + p * Ws, true, EDGE ? kk + 1 < Wi : true);
            if (p & 1)
                step(V, sb, sa);
            else
                step(V, sa, sb);
        }
        ptr += PF * Ws;
    }
    for (; s < nm; s += PF) {
#pragma unroll
        for (int p = 0; p < PF; ++p) {
            if (s + p < nm) {
                const uint32_t V = quant_in(raw[p]);
                fetch(s + p + PF + 1, ptr + p * Ws, raw[p]);
                if (p & 1)
                    step(V, sb, sa);
                else
                    step(V, sa, sb);
            }
        }
        ptr += PF * Ws;
    }
    if (nm < n) {  // at most one step: the absent row H
        if (nm & 1)
            step(S2, sb, sa);
        else
            step(S2, sa, sb);
    }
}

// Work: per image, lattice rows [v0, v1) in row blocks of L2L_RB, x column
// tiles; unit = one (tile, row) and the order (row block, tile, row), so the
// warps of a CTA hold adjacent tiles of the same rows.  All images' units
// form one range cut evenly over the CTAs; inside a CTA each image's share is
// cut evenly over the 16 warps, then the CTA folds that image's bins into
// hist[image] (one __syncthreads pair per image).
// PF / MINB: rows in flight per lane / CTAs per SM the registers are
// budgeted for -- 8 / 1 for single images (latency-bound: more bytes in
// flight per warp), 6 / 2 for batches (measured: profiles/r01/lines2d_notes.md, profiles/r02/s5/NOTES.md).
template <int DT, int QM, bool VEC, int PF, int MINB, int WS>
__global__ void __launch_bounds__(L2L_NTH, MINB) lines2d_kernel(const typename Elem<DT>::T* __restrict__ buf, LGeo g,
                                                             QuantDev q, unsigned long long* __restrict__ hist)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    char* h = reinterpret_cast<char*>(smem_raw);
    const int M2 = g.M + 2;
    const int hs = g.hs;
    const LLay lay = lines_layout(hs, L2L_SIG, g.M);
    float* tt = reinterpret_cast<float*>(h + lay.tt);
    uint32_t* hw = reinterpret_cast<uint32_t*>(h);
    for (int i = threadIdx.x; i < lay.end / 4; i += blockDim.x) hw[i] = 0;
    __syncthreads();
    if (QM != FT_Q_IDENTITY && QM != FT_Q_POW2 && QM != FT_Q_UMAGIC)
        for (int i = threadIdx.x; i < M2; i += blockDim.x) tt[i] = q.tt[i];
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t topd = sb + (uint32_t)lay.dtop, topp = sb + (uint32_t)lay.ptop;
    constexpr int NW = L2L_NTH / 32;
    const int64_t nrows = g.v1 - g.v0;
    const int ntiles = g.tiles_k;
    const int64_t Timg = cdiv(nrows, (int64_t)L2L_RB) * ntiles * L2L_RB;
    const int64_t batch = g.n_items;  // images
    const int64_t total = batch * Timg;
    const int64_t U0 = total * blockIdx.x / gridDim.x, U1 = total * (blockIdx.x + 1) / gridDim.x;
    // bins grow downward from the region tops: level l sits l + 1 words below
    const int rw = hs / 4, dt = lay.dtop / 4, pt = lay.ptop / 4, mt = pt - LINES_MINUS / 4;
    for (int64_t b = U0 / Timg; b < batch && b * Timg < U1; ++b) {
        const int64_t a = max(U0, b * Timg) - b * Timg, e = min(U1, (b + 1) * Timg) - b * Timg;
        const int64_t wa = a + (e - a) * warp / NW, we = a + (e - a) * (warp + 1) / NW;
        const typename Elem<DT>::T* img = buf + b * g.bstride;
        for (int64_t u = wa; u < we;) {
            const int64_t piece = u / L2L_RB;
            const int r = (int)(u - piece * L2L_RB);
            const int64_t len = min(we - u, (int64_t)(L2L_RB - r));
            u += len;
            const int64_t rb = piece / ntiles;
            const int t = (int)(piece - rb * ntiles);
            const int64_t r0 = rb * L2L_RB + r, r1 = min(r0 + len, nrows);
            if (r0 >= r1) continue;
            const int k0 = t * 62 - 1;
            if (k0 >= 1 && k0 + 63 <= g.W)
                lines2d_item<DT, QM, VEC, false, PF, WS>(img, g, q, tt, topd, topp, g.v0 + r0, g.v0 + r1, k0, lane);
            else
                lines2d_item<DT, QM, VEC, true, PF, WS>(img, g, q, tt, topd, topp, g.v0 + r0, g.v0 + r1, k0, lane);
        }
        __syncthreads();
        // fold: C = sum of signature rows, E = sum (4 - u) rows, EC = plus -
        // minus - sum s rows, V = EC + E - C
        unsigned long long* out = hist + b * 4 * M2;
        for (int l = threadIdx.x; l < M2; l += blockDim.x) {
            uint32_t c = 0, ed = 0;
            int32_t ec = (int32_t)(hw[pt - (l + 1)] - hw[mt - (l + 1)]);
            hw[pt - (l + 1)] = 0;
            hw[mt - (l + 1)] = 0;
#pragma unroll
            for (int s = 0; s < L2L_SIG; ++s) {
                const uint32_t v = hw[dt - s * rw - (l + 1)];
                hw[dt - s * rw - (l + 1)] = 0;
                c += v;
                ed += (uint32_t)(4 - s % 5) * v;
                ec -= (s / 5 - 1) * (int32_t)v;
            }
            const int64_t vx = (int64_t)ec + (int64_t)ed - (int64_t)c;
            if (c) atomicAdd(&out[l], (unsigned long long)c);
            if (ed) atomicAdd(&out[M2 + l], (unsigned long long)ed);
            if (vx) atomicAdd(&out[2 * M2 + l], (unsigned long long)vx);
        }
        __syncthreads();
    }
}

// 16-bit packed signature offsets: 14 hs + (M + 1) * 4 + base must fit
static int lines2d_hs(int M) { return 255 * (int)cdiv(cdiv((int64_t)(M + 2) * 4, 255), 4) * 4; }
static bool lines2d_ok(int M) { return lines_layout_ok(lines2d_hs(M), L2L_SIG, M); }

template <int DT, int QM>
static int launch_lines2d(const ft_window* win, int64_t H, int64_t W, int64_t v0, int64_t v1, const ft_quant* qa,
                          int32_t M, uint64_t* hist, cudaStream_t st)
{
    using T = typename Elem<DT>::T;
    LGeo g{};
    g.H = H; g.W = W; g.D = 1; g.v0 = v0; g.v1 = v1; g.first = win->first; g.M = M;
    g.bstride = win->batch_stride;
    g.hs = lines2d_hs(M);
    g.hk = g.hs / 255;
    g.four = 4;
    g.tiles_k = (int)((W + 1) / 62 + 1);  // tile t: lattice columns 62 t - 1 .. 62 t + 60
    g.n_items = std::max<int64_t>(win->batch, 1);
    const bool vec = W % 2 == 0 && (g.n_items <= 1 || win->batch_stride % 2 == 0) &&
                     reinterpret_cast<uintptr_t>(win->data) % (2 * sizeof(T)) == 0;
    QuantDev qd = qdev(qa);
    if (QM == FT_Q_POW2) qd.inv = M > 0 ? qd.scale / (float)M : 0.f;
    if (QM == FT_Q_UMAGIC && !umagic_fill(qa, M, DT == FT_U8 ? 256 : 65536, qd)) return FT_ERR_INTERNAL;
    const size_t smem = (size_t)lines_layout(g.hs, L2L_SIG, M).end;
    using K = void (*)(const T*, LGeo, QuantDev, unsigned long long*);
    const bool single = g.n_items == 1;
    K kern = single ? (vec ? lines2d_kernel<DT, QM, true, 8, 1, 0> : lines2d_kernel<DT, QM, false, 8, 1, 0>)
                    : (vec ? lines2d_kernel<DT, QM, true, L2B_PF, L2B_MINB, 0> : lines2d_kernel<DT, QM, false, L2B_PF, L2B_MINB, 0>);
    // the BASELINE configs' row lengths (C2: 8192 f32 pow2, C3: 1024 u8
    // identity) with immediate-offset row loads
    if constexpr ((DT == FT_F32 && QM == FT_Q_POW2) || (DT == FT_U8 && QM == FT_Q_IDENTITY)) {
        if (vec && W == 8192) kern = single ? lines2d_kernel<DT, QM, true, 8, 1, 8192> : lines2d_kernel<DT, QM, true, L2B_PF, L2B_MINB, 8192>;
        if (vec && W == 1024) kern = single ? lines2d_kernel<DT, QM, true, 8, 1, 1024> : lines2d_kernel<DT, QM, true, L2B_PF, L2B_MINB, 1024>;
    }
    FT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    FT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, L2L_NTH, smem));
    if (per_sm < 1) return FT_ERR_ARG;
    const int64_t units = g.n_items * cdiv(v1 - v0, (int64_t)L2L_RB) * g.tiles_k * L2L_RB;
    // >= one piece per warp per CTA
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)nsm_l() * per_sm,
                                                                cdiv(units, (int64_t)(L2L_NTH / 32) * L2L_RB)));
    kern<<<(int)grid, L2L_NTH, smem, st>>>(static_cast<const T*>(win->data), g, qd,
                                          reinterpret_cast<unsigned long long*>(hist));
    FT_CUDA_TRY(cudaGetLastError());
    return FT_OK;
}

}  // namespace ft

#ifndef FT_DEV_KERNEL_ONLY
using namespace ft;

extern "C" int ft_lines2d(const ft_window* win, int64_t H, int64_t W, int64_t v0, int64_t v1, const ft_quant* q,
                          int32_t M, uint64_t* hist, void* stream)
{
    if (!win || !hist || H < 1 || W < 1 || M < 0 || v0 < 0 || v1 > H + 1 || v0 > v1) return FT_ERR_ARG;
    if (!lines2d_ok(M)) return FT_ERR_ARG;
    if (win->batch > 1 && win->batch_stride < win->count * W) return FT_ERR_ARG;
    if (v0 == v1) return FT_OK;
    if (!window_ok(win, H, v0, v1, 2)) return FT_ERR_ARG;
    const int qm = effective_qmode(q, true);
    if (qm != FT_Q_IDENTITY && !q->thresholds) return FT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    QuantDev probe{};
    switch (win->dtype) {
    case FT_I32:
        if (qm != FT_Q_IDENTITY) return FT_ERR_ARG;
        return launch_lines2d<FT_I32, FT_Q_IDENTITY>(win, H, W, v0, v1, q, M, hist, st);
    case FT_U8:
        if (qm == FT_Q_IDENTITY) return launch_lines2d<FT_U8, FT_Q_IDENTITY>(win, H, W, v0, v1, q, M, hist, st);
        if (umagic_fill(q, M, 256, probe)) return launch_lines2d<FT_U8, FT_Q_UMAGIC>(win, H, W, v0, v1, q, M, hist, st);
        if (qm == FT_Q_TABLE || qm == FT_Q_POW2) return launch_lines2d<FT_U8, FT_Q_TABLE>(win, H, W, v0, v1, q, M, hist, st);
        return launch_lines2d<FT_U8, FT_Q_TABLE_ROBUST>(win, H, W, v0, v1, q, M, hist, st);
    case FT_U16:
        if (qm == FT_Q_IDENTITY) return launch_lines2d<FT_U16, FT_Q_IDENTITY>(win, H, W, v0, v1, q, M, hist, st);
        if (umagic_fill(q, M, 65536, probe)) return launch_lines2d<FT_U16, FT_Q_UMAGIC>(win, H, W, v0, v1, q, M, hist, st);
        if (qm == FT_Q_POW2) return launch_lines2d<FT_U16, FT_Q_POW2>(win, H, W, v0, v1, q, M, hist, st);
        if (qm == FT_Q_TABLE) return launch_lines2d<FT_U16, FT_Q_TABLE>(win, H, W, v0, v1, q, M, hist, st);
        return launch_lines2d<FT_U16, FT_Q_TABLE_ROBUST>(win, H, W, v0, v1, q, M, hist, st);
    case FT_F32:
        if (qm == FT_Q_IDENTITY) return FT_ERR_ARG;
        if (qm == FT_Q_POW2) return launch_lines2d<FT_F32, FT_Q_POW2>(win, H, W, v0, v1, q, M, hist, st);
        if (qm == FT_Q_TABLE) return launch_lines2d<FT_F32, FT_Q_TABLE>(win, H, W, v0, v1, q, M, hist, st);
        return launch_lines2d<FT_F32, FT_Q_TABLE_ROBUST>(win, H, W, v0, v1, q, M, hist, st);
    }
    return FT_ERR_ARG;
}

extern "C" int ft_lines2d_ok(int32_t M) { return M >= 0 && lines2d_ok(M) ? 1 : 0; }
#endif  // FT_DEV_KERNEL_ONLY
