// ft_lines3d.cuh -- fused EC / surface-area / volume histograms of 3D fields by
// line decomposition: the curve path of the north star.
//
// The reference builds the EC curve from per-vertex transition counts
// (contrib3d.py:241-348) and folds them with the weight tables
// (descriptors.py:169-178).  ft_lattice.cu restates the same curves as
// element counts by level (EC_26C = V - E + F - C, surface = 2F - 6C,
// volume = C); this kernel needs far fewer histogram events for them:
//
// * Slicing the closed cubical complex along k and then j (inclusion-
//   exclusion of closed sets, the open slab between two planes counts with
//   chi = -1) gives  chi_3D = sum over i-lines of
//       chi1(A) - chi1(B) - chi1(C) + chi1(D),
//   A = cell levels, B = min over (j-1, j), C = min over (k-1, k), D = min over
//   both, every family on the lattice positions (j, k) in [0, W] x [0, D].  A
//   1D line of unit intervals has chi1 = sum over its cells of +1 (local min
//   along i) / -1 (local max), so EC events are SPARSE: ~10% of cells per
//   family on the benchmark fields, booked with dummy-address
//   shared atomics (lanes without an event all hit one merged word).
// * Cubes and faces are booked once per cell by their per-cell signature, as
//   in lattice3d_sig_kernel: the row u = #face neighbours activating before
//   the cell (so F = sum (6 - u)), and -- when the 16-bit row offsets allow
//   (FOLD) -- the cell's own A-line event s_i in {-1, 0, +1} (row
//   u + 7 (s_i + 1)), so family A costs no extra atomic.
//
// Ties follow one strict order per family: lower i first along a line, and
// the reference-style (level, index) order for face ownership.  Every
// choice gives the same counts by level, so the curves are bit-exact
// (tests/test_gpu_lattice.py against the reference golden curves and the
// pinned oracle).
//
// Per lattice point: 2 dense shared atomics per cell pair (signature) + ~0.6
// sparse ones, against 10 dense for lattice3d_rb_kernel -- the shared-memory
// pipe (95% busy there) stops being the limiter.  Same warp-strip register
// march as lattice3d_rb_kernel (no staging, no CTA barrier).  Interior warp
// strips run a guard-free loop (no load predicates, no sentinel selects, and
// the FT_Q_POW2 quantizer is FMUL.SAT + FFMA2.RM + FADD2.RM, no F2I).
//
// Output rows (uint64 [3][M+2], accumulated): cells C, faces F, and
// X = V - E = EC - F + C (two's complement; X may be negative).
//
// The kernel templates live here; ft_lines.cu holds the C entry points and
// the per-input-type launchers are instantiated in ft_lines_f32p.cu (the
// benchmark path: f32, power-of-two range), ft_lines_f32t.cu, ft_lines_u16.cu
// and ft_lines_u8i32.cu, so that nvcc compiles them in parallel.
#pragma once
#include "ft_lines.cuh"

namespace ft {

#ifndef LINES_NTH_DEF
#define LINES_NTH_DEF 512
#endif
#ifndef LINES_MINB_DEF
#define LINES_MINB_DEF 1
#endif
constexpr int LINES_NTH = LINES_NTH_DEF;    // warp strips per CTA item = LINES_NTH / 32
constexpr int LINES_MINB = LINES_MINB_DEF;  // CTAs per SM the registers are budgeted for
#ifndef LINES_R_DEF
#define LINES_R_DEF 4
#endif
constexpr int LINES_R = LINES_R_DEF;    // lattice rows per warp strip

__host__ __device__ inline int lines_nsig(bool fold) { return fold ? 21 : 7; }

// One warp strip (R lattice rows x 62 lattice columns) marching the planes of
// a chunk [ia, ib).  Shared memory (lines_layout): the signature rows below
// topd, the plus / minus rows of the EC events of the B/C/D lines (and of the
// A lines unless FOLD) below topp (topd / topp: shared addresses).
// EDGE 0: interior strip (no guards); 1: every row present, columns outside
// the field (clamped loads, masked halves); 2: rows and columns guarded.
template <int DT, int QM, bool VEC, int R, bool FOLD, int DS, int EDGE>
__device__ __forceinline__ void lines_item(const typename Elem<DT>::T* __restrict__ buf, const LGeo& g,
                                           const QuantDev& q, const float* __restrict__ tt, uint32_t topd_u,
                                           uint32_t topp_u, int64_t ia, int64_t ib, int j0, int k0, int lane)
{
    using P2 = typename Pair<DT>::T;
    using T = typename Elem<DT>::T;
    constexpr int NR = R + 2;  // cell rows j0-1 .. j0+R held per plane
    constexpr uint32_t FULL = 0xFFFFFFFFu;
    // DS > 0: the row stride D as a compile-time constant, so the NR row loads
    // of a plane use immediate offsets from one pointer (no address math)
    const int Di = DS > 0 ? DS : (int)g.D;
    const int64_t pe = g.W * (int64_t)Di;
    const uint32_t sent4 = (uint32_t)(g.M + 1) * 4u;
    constexpr uint32_t sbw = LINES_REL0;         // packed words: (level + 1) * 4 per half
    const uint32_t S2 = sent4 * 0x10001u + sbw;  // sentinel level word
    const uint32_t sent_lv2 = (uint32_t)(g.M + 1) * 0x10001u;
    const uint32_t hk = (uint32_t)g.hk;  // signature row stride / 255
    const float Mf = (float)g.M;
    // lane l holds cells kk, kk+1 (kk even: aligned pair loads); lattice
    // columns k0 .. k0+61 are computed by lane 0's high half, both halves of
    // lanes 1 .. 30 and lane 31's low half (the other two halves are the halo:
    // lane 0's low cell feeds the -k neighbour, lane 31's high cell the +k one)
    const int kk = k0 - 1 + 2 * lane;
    // through a shuffle so that ptxas keeps a mask register (one 3-input LOP3)
    // instead of SEL on a predicate
    const uint32_t lmask = __shfl_sync(FULL, lane == 0 ? 0xFFFF0000u : lane == 31 ? 0x0000FFFFu : FULL, lane);
    const uint32_t lsel = __shfl_sync(FULL, lane_sel(lane), lane);  // dense events: halo halves -> the dummy word
    // the region tops as per-lane registers (through a shuffle: as uniform
    // values ptxas re-materialises them with a move in front of every IDP)
    const uint32_t topd = __shfl_sync(FULL, topd_u, lane), topp = __shfl_sync(FULL, topp_u, lane);
    const int n = (int)(ib - ia);

    // Absent cells (outside the field) read as the sentinel:
    // * planes t = -1 .. n (plane ia-1+t) exist iff t_lo <= t < t_hi (warp-
    //   uniform; only the first two and the last plane of the field);
    // * EDGE strips (at the k boundary) load CLAMPED in-row pairs (always
    //   valid memory) and mask absent cells per 16-bit half (lanekeep); at the
    //   j boundary (EDGE 2) they also predicate / overwrite absent rows.
    //   Interior strips do none of it.
    const int t_lo = (int)max((int64_t)-1, 1 - ia);
    const int t_hi = (int)min((int64_t)(n + 2), g.H - ia + 1);
    // planes t < tf are fetched (the window holds planes ia-2 .. ib-1 only)
    const int tf = min(n + 1, t_hi);
    const bool okx = kk >= 0 && kk < (int)g.D, oky = kk + 1 >= 0 && kk + 1 < (int)g.D;
    const uint32_t lanekeep = (okx ? 0x0000FFFFu : 0u) | (oky ? 0xFFFF0000u : 0u);
    const int kc = EDGE == 0 ? kk : VEC ? min(max(kk, 0), (int)g.D - 2) : min(max(kk, 0), (int)g.D - 1);
    uint32_t rowok = (1u << NR) - 1u;
    if constexpr (EDGE == 2) {
        rowok = 0;
#pragma unroll
        for (int r = 0; r < NR; ++r) rowok |= (j0 - 1 + r >= 0 && j0 - 1 + r < (int)g.W) ? 1u << r : 0u;
    }
    // word of row 0 in plane ia-2 (t = -1)
    const T* ptr = buf + ((ia - 2 - g.first) * pe + (int64_t)(j0 - 1) * Di + kc);

    auto fetch = [&](int t, const T* at, P2(&dst)[NR]) {
        if (t >= t_lo && t < tf) {
            if constexpr (EDGE == 2) {
#pragma unroll
                for (int r = 0; r < NR; ++r)
                    if ((rowok >> r) & 1u) dst[r] = load_pair<DT, VEC>(at + r * Di, true, kk + 1 < (int)g.D);
            } else if constexpr (EDGE == 1) {
#pragma unroll
                for (int r = 0; r < NR; ++r) dst[r] = load_pair<DT, VEC>(at + r * Di, true, kk + 1 < (int)g.D);
            } else {
#pragma unroll
                for (int r = 0; r < NR; ++r) dst[r] = load_pair<DT, VEC>(at + r * Di, true, true);
            }
        }
    };
    // quantize a plane known to exist
    auto quant_in = [&](const P2(&src)[NR], uint32_t(&V)[NR]) {
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            uint32_t v;
            if constexpr (QM == FT_Q_POW2)
                v = pack_pow2_sat<DT>(src[r], q.inv, Mf, g.four, sbw);
            else if constexpr (QM == FT_Q_UMAGIC)
                v = pack_pair_umagic<DT>(src[r], q, g.four, sbw);
            else if constexpr (QM == FT_Q_IDENTITY && (DT == FT_U8 || DT == FT_U16))
                v = pack_pair_ident<DT>(src[r], sent_lv2, g.four, sbw);
            else
                v = pack_pair<DT, QM, 0>(src[r], true, true, tt, q, g.M, sent4) + sbw;
            V[r] = EDGE ? sel_mask(lanekeep, v, S2) : v;
        }
        if constexpr (EDGE == 2) {
#pragma unroll
            for (int r = 0; r < NR; ++r)
                if (!((rowok >> r) & 1u)) V[r] = S2;
        }
    };
    auto quant = [&](int t, const P2(&src)[NR], uint32_t(&V)[NR]) {
        if (t >= t_lo && t < t_hi) {
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                uint32_t v;
                if constexpr (QM == FT_Q_POW2)
                    v = pack_pow2_sat<DT>(src[r], q.inv, Mf, g.four, sbw);
                else if constexpr (QM == FT_Q_UMAGIC)
                    v = pack_pair_umagic<DT>(src[r], q, g.four, sbw);
                else if constexpr (QM == FT_Q_IDENTITY && (DT == FT_U8 || DT == FT_U16))
                    v = pack_pair_ident<DT>(src[r], sent_lv2, g.four, sbw);
                else
                    v = pack_pair<DT, QM, 0>(src[r], true, true, tt, q, g.M, sent4) + sbw;
                V[r] = EDGE ? sel_mask(lanekeep, v, S2) : v;
            }
            if constexpr (EDGE == 2) {
#pragma unroll
                for (int r = 0; r < NR; ++r)
                    if (!((rowok >> r) & 1u)) V[r] = S2;
            }
        } else {
#pragma unroll
            for (int r = 0; r < NR; ++r) V[r] = S2;
        }
    };
    // k-shifted words and the min-derived families of one plane
    auto derive = [&](const uint32_t(&V)[NR], uint32_t(&Wm)[NR], uint32_t(&C)[NR]) {
#pragma unroll
        for (int r = 0; r <= R; ++r) {
            Wm[r] = shift_pair(__shfl_up_sync(FULL, V[r], 1), V[r]);
            C[r] = vmin2(V[r], Wm[r]);
        }
    };

    // march state of the previous cell plane; two copies, written alternately
    // by the 2-step unrolled march, so no register moves carry it over
    struct St {
        uint32_t pV[NR], pt3[R + 1], pWm[R + 1];  // pt3: the +i term t3 of plane p-2 (tmi = 255 - pt3)
        uint32_t pB[R + 1], eB[R + 1], pC[R + 1], eC[R + 1], pD[R + 1], eD[R + 1];
    };
    St sa, sb2;
    P2 ra[NR], rb[NR];  // two planes in flight per lane
    {
        fetch(-1, ptr, ra);
        fetch(0, ptr + pe, rb);
        uint32_t V0[NR], Wm0[NR], C0[NR], Wm1[NR], C1[NR];
        quant(-1, ra, V0);       // plane ia-2
        quant(0, rb, sa.pV);     // plane ia-1
        derive(V0, Wm0, C0);
        derive(sa.pV, Wm1, C1);
#pragma unroll
        for (int r = 1; r <= R; ++r) {
            sa.pt3[r] = hff(cmp2(V0[r], sa.pV[r])) ^ FF2;  // plane ia-1's -i neighbour NOT first
            sa.pWm[r] = Wm1[r];
            const uint32_t b0 = vmin2(V0[r - 1], V0[r]), b1 = vmin2(sa.pV[r - 1], sa.pV[r]);
            const uint32_t d0 = vmin2(C0[r - 1], C0[r]), d1 = vmin2(C1[r - 1], C1[r]);
            sa.pB[r] = b1;
            sa.eB[r] = cmp2(b0, b1);
            sa.pC[r] = C1[r];
            sa.eC[r] = cmp2(C0[r], C1[r]);
            sa.pD[r] = d1;
            sa.eD[r] = cmp2(d0, d1);
        }
    }
    fetch(1, ptr + 2 * pe, ra);
    fetch(2, ptr + 3 * pe, rb);
    ptr += 4 * pe;  // next fetch: t = 3

    // One step: plane t (cell plane p = ia-1+t) arrives in V; every event of
    // cell plane p-1 (whose +i neighbours are now known) is booked.  o = the
    // state of plane p-1, x receives the state of plane p.
    auto step = [&](const uint32_t(&V)[NR], const St& o, St& x) {
        uint32_t Wm[NR], C[NR];
        derive(V, Wm, C);
        uint32_t tpj = 0;
#pragma unroll
        for (int r = 1; r <= R; ++r) {
            const uint32_t W_ = V[r];
            // signature of the plane-(p-1) cell: "face neighbour n activates
            // first" = bit 15 / 31 of c' - n + k (k = 0 for -side, -1 for +side)
            const uint32_t cb = o.pV[r] | 0x80008000u;
            const uint32_t t2 = hff(cb - o.pWm[r]);                 // -k
            const uint32_t t3 = hff(cb - W_ - 0x10001u);            // +i
            const uint32_t t4 = hff(cb - o.pV[r + 1] - 0x10001u);   // +j
            // -j: row 1 compares with the halo row; row r > 1 is the
            // complement of row r-1's +j term (t1 = 255 - tpj)
            // +k: "right neighbour first" is the complement of the right
            // neighbour's -k term (lo: this word's hi half, hi: the next lane's lo)
            const uint32_t sh5 = shift_pair(t2, __shfl_down_sync(FULL, t2, 1));
            uint32_t evS;
            if constexpr (FOLD) {
                // row u + 7 (s_i + 1) = (t1 + t2 + t4 + t5) + 14 - 6 (tmi + t3) in
                // units of 255, with t5 = 255 - sh5, tmi = 255 - pt3, t1 as
                // above: plain packed adds (IADD3), the constants folded.  The
                // sums are linear and every half ENDS in [0, 20 * 255], so
                // intermediate cross-half borrows cancel.
                const uint32_t base = r == 1 ? hff(cb - o.pV[0]) + 9u * FF2 : 10u * FF2 - tpj;
                const uint32_t row = base + t2 + t4 - sh5 + 6u * (o.pt3[r] - t3);
                evS = row * hk + o.pV[r];
            } else {
                const uint32_t t1 = r == 1 ? hff(cb - o.pV[0]) : FF2 - tpj;
                const uint32_t tmi = o.pt3[r] ^ FF2;
                evS = (tmi + t1 + t2 + t3 + t4 + (FF2 - sh5)) * hk + o.pV[r];
                // A line event iff both or neither i-neighbour is first; minus (max) iff t3
                const uint32_t fA = ~(tmi ^ t3) & lmask;
                const uint32_t aA = o.pV[r] | ((t3 << 8) & 0x80008000u);
                sinc2(aA, ev_sel(fA << 8), topp);
            }
            sinc2(evS, lsel, topd);
            // B / C / D lines: event iff the along-i order flips at p-1; sign -1
            // (B, C): local min -> minus row; sign +1 (D): local max -> minus row
            const uint32_t B = vmin2(V[r - 1], W_);
            const uint32_t D = vmin2(C[r - 1], C[r]);
            const uint32_t nB = cmp2(o.pB[r], B), nC = cmp2(o.pC[r], C[r]), nD = cmp2(o.pD[r], D);
            sinc2(o.pB[r] | (nB & 0x80008000u), ev_sel((o.eB[r] ^ nB) & lmask), topp);
            sinc2(o.pC[r] | (nC & 0x80008000u), ev_sel((o.eC[r] ^ nC) & lmask), topp);
            sinc2(o.pD[r] | (~nD & 0x80008000u), ev_sel((o.eD[r] ^ nD) & lmask), topp);
            x.pt3[r] = t3;
            tpj = t4;
            x.pWm[r] = Wm[r];
            x.pB[r] = B;
            x.eB[r] = nB;
            x.pC[r] = C[r];
            x.eC[r] = nC;
            x.pD[r] = D;
            x.eD[r] = nD;
        }
#pragma unroll
        for (int r = 0; r < NR; ++r) x.pV[r] = V[r];
    };

    // steps s < nm see an existing plane t = s+1; only the last step of the
    // field's last chunk (plane H) can follow, with a sentinel plane
    uint32_t V[NR];
    const int nm = min(n, t_hi - 1);
    int s = 0;
    for (; s < nm; s += 2) {
        quant_in(ra, V);  // plane t = s+1
        if (s + 3 < tf) fetch(s + 3, ptr, ra);
        ptr += pe;
        step(V, sa, sb2);
        if (s + 1 >= nm) {
            ++s;
            break;
        }
        quant_in(rb, V);
        if (s + 4 < tf) fetch(s + 4, ptr, rb);
        ptr += pe;
        step(V, sb2, sa);
    }
    if (s < n) {  // at most one step: the absent plane H
#pragma unroll
        for (int r = 0; r < NR; ++r) V[r] = S2;
        if (s & 1)
            step(V, sb2, sa);
        else
            step(V, sa, sb2);
    }
}

// The CTA tiles (TJ = 16 R rows x 62 columns) of ntk column tiles, rows up to
// the last tile holding an interior strip, times the planes.  Full rounds:
// CTA b marches tile r G + b over every plane (the G CTAs of a round hold
// adjacent tiles at about the same planes, so the halo rows and the partial
// 32-byte sectors at tile edges are read from DRAM once and hit L2 for the
// neighbour).  The leftover tiles x planes are cut evenly over the CTAs
// (tile-major segments of consecutive planes), so no CTA waits on a quantised
// item count.  Warp strips with rows outside 1 .. W-1 are left to the warp
// loop.  f(j0, column tile, ia, ib).
template <int R, typename F>
__device__ __forceinline__ void cta_tiles(const LGeo& g, int ntk, int64_t np, int warp, F&& f)
{
    constexpr int TJ = (LINES_NTH / 32) * R;
    const int G = gridDim.x, b = blockIdx.x;
    const int ntiles = g.tiles_j * ntk;
    const int rounds = ntiles / G;
    auto seg = [&](int tile, int64_t p0, int64_t p1) {
        const int tj = tile / ntk;
        const int j0 = tj * TJ + warp * R;
        if (j0 >= 1 && j0 + R < g.W) f(j0, tile - tj * ntk, g.v0 + p0, g.v0 + p1);
    };
    for (int r = 0; r < rounds; ++r) seg(r * G + b, 0, np);
    const int64_t T = (int64_t)(ntiles - rounds * G) * np;
    const int64_t u_end = T * (b + 1) / G;
    for (int64_t u = T * b / G; u < u_end;) {
        const int t = (int)(u / np);
        const int64_t p = u - (int64_t)t * np;
        const int64_t len = min(u_end - u, np - p);
        u += len;
        seg(rounds * G + t, p, p + len);
    }
}

// Work split.  MODE 0 / 2: (A) the CTA tiles of the interior column tiles
// (guard-free march), then (B) those of the k-boundary column tiles (column-
// guarded march), each cut evenly over the CTAs (cta_tiles).  MODE 1 / 2: (C)
// the row-boundary strips, one warp per strip-chunk (fully guarded march).
// Separate loops, separate instantiations of lines_item: the boundary code
// costs the interior march no instructions or registers.
template <int DT, int QM, bool VEC, int R, bool FOLD, int DS, int MODE>
__global__ void __launch_bounds__(LINES_NTH, LINES_MINB) lines3d_kernel(const typename Elem<DT>::T* __restrict__ buf,
                                                                        LGeo g, QuantDev q,
                                                                        unsigned long long* __restrict__ hist)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    char* h = reinterpret_cast<char*>(smem_raw);
    const int M2 = g.M + 2;
    const int hs = g.hs;
    const LLay lay = lines_layout(hs, lines_nsig(FOLD), g.M);
    float* tt = reinterpret_cast<float*>(h + lay.tt);  // threshold table: in the minus/plus gap
    for (int i = threadIdx.x; i < lay.end / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(h)[i] = 0;
    __syncthreads();  // the table lies inside the zeroed range
    if (QM != FT_Q_IDENTITY && QM != FT_Q_POW2 && QM != FT_Q_UMAGIC)
        for (int i = threadIdx.x; i < M2; i += blockDim.x) tt[i] = q.tt[i];
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x / 32;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t topd = sb + (uint32_t)lay.dtop, topp = sb + (uint32_t)lay.ptop;
    if constexpr (MODE != 1) {
        // A: interior column tiles; B: the k-boundary ones (EDGE 1 march)
        const int64_t np = g.v1 - g.v0;
        const int ntk = g.tiles_k - g.kb_lo - g.kb_hi;
        cta_tiles<R>(g, ntk, np, warp, [&](int j0, int tk, int64_t ia, int64_t ib) {
            lines_item<DT, QM, VEC, R, FOLD, DS, 0>(buf, g, q, tt, topd, topp, ia, ib, j0, (g.kb_lo + tk) * 62 - 1, lane);
        });
        cta_tiles<R>(g, g.kb_lo + g.kb_hi, np, warp, [&](int j0, int tk, int64_t ia, int64_t ib) {
            const int t = tk < g.kb_lo ? tk : g.tiles_k - g.kb_hi + (tk - g.kb_lo);
            lines_item<DT, QM, VEC, R, FOLD, DS, 1>(buf, g, q, tt, topd, topp, ia, ib, j0, t * 62 - 1, lane);
        });
    }
    if constexpr (MODE != 0) {
        // C: the row-boundary strips (rf_j0: j0 = 0 and the strips reaching
        // row W-1 or past it) of every column tile
        const int64_t nw = (int64_t)gridDim.x * (LINES_NTH / 32);
        const int64_t per_chunk = (int64_t)g.tiles_k * g.rf_n;
        for (int64_t it = (int64_t)blockIdx.x * (LINES_NTH / 32) + warp; it < g.e_items; it += nw) {
            const int64_t ch = it / per_chunk;
            const int rem = (int)(it - ch * per_chunk);
            const int tk = rem / g.rf_n;
            const int j0 = g.rf_j0[rem - tk * g.rf_n];
            const int64_t ia = g.v0 + ch * g.e_chunk;
            const int64_t ib = min(ia + (int64_t)g.e_chunk, g.v1);
            lines_item<DT, QM, VEC, R, FOLD, DS, 2>(buf, g, q, tt, topd, topp, ia, ib, j0, tk * 62 - 1, lane);
        }
    }
    __syncthreads();
    // fold: C = sum of signature rows, F = sum (6 - u) rows, EC = A events (row
    // groups, or plus/minus when !FOLD) + plus - minus, X = EC - F + C
    // (bins grow downward from the region tops: level l sits l + 1 words below)
    const uint32_t* hw = reinterpret_cast<const uint32_t*>(h);
    const int rw = hs / 4, dt = lay.dtop / 4, pt = lay.ptop / 4;
    for (int l = threadIdx.x; l < M2; l += blockDim.x) {
        uint32_t c = 0, f = 0;
        int32_t ec = (int32_t)(hw[pt - (l + 1)] - hw[pt - LINES_MINUS / 4 - (l + 1)]);
#pragma unroll
        for (int s = 0; s < lines_nsig(FOLD); ++s) {
            const uint32_t v = hw[dt - s * rw - (l + 1)];
            c += v;
            f += (uint32_t)(6 - s % 7) * v;
            if (FOLD) ec += (s / 7 - 1) * (int32_t)v;
        }
        const int64_t x = (int64_t)ec - (int64_t)f + (int64_t)c;
        if (c) atomicAdd(&hist[l], (unsigned long long)c);
        if (f) atomicAdd(&hist[M2 + l], (unsigned long long)f);
        if (x) atomicAdd(&hist[2 * M2 + l], (unsigned long long)x);
    }
}

// signature rows are 255 K bytes apart (K a multiple of 4: word-aligned rows)
static int lines_hs(int M) { return 255 * (int)cdiv(cdiv((int64_t)(M + 2) * 4, 255), 4) * 4; }
// 16-bit packed bin offsets (lines_layout_ok): 21 rows with the folded A-line
// events, else 7 rows + the A events in the plus / minus rows
static bool lines_fold_ok(int M, int hs) { return lines_layout_ok(hs, 21, M); }
static bool lines_ok(int M) { return lines_layout_ok(lines_hs(M), 7, M); }


// Interior and boundary items in one launch (MODE 2)
template <int DT, int QM, bool VEC, bool FOLD, int DS, int MODE>
static int launch_lines_kernel(const ft_window* win, LGeo g, const QuantDev& qd, size_t smem, uint64_t* hist,
                               cudaStream_t st)
{
    using T = typename Elem<DT>::T;
    auto kern = lines3d_kernel<DT, QM, VEC, LINES_R, FOLD, DS, MODE>;
    FT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    FT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, LINES_NTH, smem));
    if (per_sm < 1) return FT_ERR_ARG;
    const int64_t cap = (int64_t)nsm_l() * per_sm;
    // CTA tiles: column tiles x row tiles up to the last interior strip
    // (j0 + R < W); k-boundary column tiles: k0 < 1 (tile 0), k0 + 63 > D
    constexpr int TJ = (LINES_NTH / 32) * LINES_R;
    g.kb_lo = 1;
    g.kb_hi = 0;
    for (int tk = g.tiles_k - 1; tk >= 1 && tk * 62 + 62 > g.D; --tk) ++g.kb_hi;
    g.tiles_j = g.W > LINES_R ? (int)((g.W - LINES_R - 1) / TJ + 1) : 0;
    const int64_t np = g.v1 - g.v0;
    const int64_t work = MODE == 1 ? 0 : (int64_t)g.tiles_j * g.tiles_k * np;
    // warp strips: j0 = 0 and every strip reaching row W-1 or past it
    g.rf_n = 0;
    for (int64_t j0 = 0; j0 <= g.W && g.rf_n < 4; j0 += LINES_R)
        if (j0 < 1 || j0 + LINES_R >= g.W) g.rf_j0[g.rf_n++] = (int)j0;
    const int64_t strips = (int64_t)g.tiles_k * g.rf_n;
    // one warp per strip-chunk, the strip-planes spread over every warp of
    // the grid (>= 8 planes per chunk): the CTA loops are evenly split, so an
    // uneven share of boundary chunks would set the kernel's tail (C4a: one
    // 65-plane chunk on 9 % of the warps cost ~20 %)
    constexpr int NWC = LINES_NTH / 32;
    const int64_t grid0 = std::max<int64_t>(1, std::min<int64_t>(cap, std::max<int64_t>(cdiv(work, 32), cdiv(strips, NWC))));
    g.e_chunk = (int)std::min<int64_t>(np, std::max<int64_t>(8, cdiv(np * strips, grid0 * NWC)));
    g.e_items = MODE == 0 ? 0 : strips * cdiv(np, g.e_chunk);
    // the CTA ranges: >= 32 tile-planes per CTA
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(cap, std::max<int64_t>(cdiv(work, 32), cdiv(g.e_items, NWC))));
    kern<<<(int)grid, LINES_NTH, smem, st>>>(static_cast<const T*>(win->data), g, qd,
                                            reinterpret_cast<unsigned long long*>(hist));
    FT_CUDA_TRY(cudaGetLastError());
    return FT_OK;
}

template <int DT, int QM, bool VEC, bool FOLD, int DS>
static int launch_lines_two(const ft_window* win, const LGeo& g, const QuantDev& qd, size_t smem, uint64_t* hist,
                            cudaStream_t st)
{
    return launch_lines_kernel<DT, QM, VEC, FOLD, DS, 2>(win, g, qd, smem, hist, st);
}

template <int DT, int QM, bool VEC, bool FOLD>
static int launch_lines_pair(const ft_window* win, const LGeo& g, const QuantDev& qd, size_t smem, uint64_t* hist,
                             cudaStream_t st)
{
    // specialised on the common row lengths of the BASELINE configs' f32 / u16
    // fields (C4a / C5 f32, C4b u16); other inputs take the generic loop
    constexpr bool spec = VEC && (DT == FT_F32 || DT == FT_U16) && QM != FT_Q_TABLE_ROBUST &&
                          !(DT == FT_U16 && QM == FT_Q_TABLE);  // u16 integer ranges run as FT_Q_UMAGIC
    if constexpr (spec) {
        switch (g.D) {
        case 2048: return launch_lines_two<DT, QM, VEC, FOLD, 2048>(win, g, qd, smem, hist, st);
        case 1024: return launch_lines_two<DT, QM, VEC, FOLD, 1024>(win, g, qd, smem, hist, st);
        case 512: return launch_lines_two<DT, QM, VEC, FOLD, 512>(win, g, qd, smem, hist, st);
        case 256: return launch_lines_two<DT, QM, VEC, FOLD, 256>(win, g, qd, smem, hist, st);
        default: break;
        }
    }
    return launch_lines_two<DT, QM, VEC, FOLD, 0>(win, g, qd, smem, hist, st);
}

template <int DT, int QM>
static int launch_lines3d(const ft_window* win, int64_t H, int64_t W, int64_t D, int64_t v0, int64_t v1,
                          const ft_quant* qa, int32_t M, uint64_t* hist, cudaStream_t st)
{
    using T = typename Elem<DT>::T;
    LGeo g{};
    g.H = H; g.W = W; g.D = D; g.v0 = v0; g.v1 = v1; g.first = win->first; g.M = M;
    g.hs = lines_hs(M);
    g.hk = g.hs / 255;
    g.four = 4;
    const bool vec = D % 2 == 0 && reinterpret_cast<uintptr_t>(win->data) % (2 * sizeof(T)) == 0;
    const bool fold = lines_fold_ok(M, g.hs);
    const size_t smem = (size_t)lines_layout(g.hs, lines_nsig(fold), M).end;
    g.tiles_k = (int)((D + 1) / 62 + 1);  // tile t: lattice columns 62 t - 1 .. 62 t + 60
    QuantDev qd = qdev(qa);
    if (QM == FT_Q_POW2) qd.inv = M > 0 ? qd.scale / (float)M : 0.f;
    if (QM == FT_Q_UMAGIC && !umagic_fill(qa, M, DT == FT_U8 ? 256 : 65536, qd)) return FT_ERR_INTERNAL;
    if (fold)
        return vec ? launch_lines_pair<DT, QM, true, true>(win, g, qd, smem, hist, st)
                   : launch_lines_pair<DT, QM, false, true>(win, g, qd, smem, hist, st);
    return vec ? launch_lines_pair<DT, QM, true, false>(win, g, qd, smem, hist, st)
               : launch_lines_pair<DT, QM, false, false>(win, g, qd, smem, hist, st);
}

// per-input-type launchers (one translation unit each)
#define FT_LINES3D_ARGS const ft_window *win, int64_t H, int64_t W, int64_t D, int64_t v0, int64_t v1, \
                        const ft_quant *q, int32_t M, uint64_t *hist, cudaStream_t st
int lines3d_f32_pow2(FT_LINES3D_ARGS);
int lines3d_f32_table(FT_LINES3D_ARGS, int qm);
int lines3d_u16(FT_LINES3D_ARGS, int qm);
int lines3d_u8i32(FT_LINES3D_ARGS, int dtype, int qm);

}  // namespace ft
