// ft_lines.cu -- fused EC / surface-area / volume histograms of 3D fields by
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
//   family on the benchmark fields, booked with predicated
//   shared atomics whose inactive lanes touch no bank.
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
// the FT_Q_POW2 quantizer is FMUL.SAT + FFMA.RM + F2I).
//
// Output rows (uint64 [3][M+2], accumulated): cells C, faces F, and
// X = V - E = EC - F + C (two's complement; X may be negative).
#include "ft_lattice.cuh"

namespace ft {

// bit 15 / 31 of x as 0 / 1 in each 16-bit half
__device__ __forceinline__ uint32_t hbit(uint32_t x) { return (x >> 15) & 0x10001u; }
// bits 15 / 31 = [prev <= cur] per 16-bit half (levels < 2^15)
__device__ __forceinline__ uint32_t cmp2(uint32_t prev, uint32_t cur) { return cur + 0x80008000u - prev; }

// Interior FT_Q_POW2 quantizer (lo = 0, hi = 2^p, M / hi exact): the reference
// clip(floor(x * M / hi + 0.5), 0, M) as sat(x / hi) (exact power-of-two
// scaling; NaN -> 0), one FMA rounded toward -inf (never crosses an integer
// upward, see to_level4) and the floor by magic addition: y + 2^23 rounded
// toward -inf is 2^23 + floor(y) for 0 <= y < 2^23, whose low mantissa bits
// ARE the level -- all on the FMA pipes (no F2I: the conversion unit is a
// quarter-rate pipe on B200).  Levels * 4, packed.
template <int DT>
__device__ __forceinline__ uint32_t pack_pow2_sat(const typename Pair<DT>::T& v, float inv, float Mf)
{
    const float a = __saturatef((float)v.x * inv);
    const float b = __saturatef((float)v.y * inv);
    const uint32_t la = __float_as_uint(__fadd_rd(__fmaf_rd(a, Mf, 0.5f), 8388608.0f));
    const uint32_t lb = __float_as_uint(__fadd_rd(__fmaf_rd(b, Mf, 0.5f), 8388608.0f));
    return __byte_perm(la, lb, 0x5410) * 4u;
}

// Shared-memory increments of both 16-bit halves of a packed address.  No
// predicates: ptxas turns predicated shared atomics into branches, so a lane
// without an event points at a DUMMY word instead (all such lanes hit the
// same word: one bank access, merged by the POPC increment).  The halves are
// split on the FMA pipe (IMAD.HI / IMAD), the ALU pipe being the busy one.
__device__ __forceinline__ void sinc2(uint32_t sbase, uint32_t addr)
{
    const uint32_t hi = __umulhi(addr, 0x10000u);
    const uint32_t lo = addr - hi * 0x10000u;
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(sbase + lo));
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(sbase + hi));
}
// halves of addr whose flag bit (15 / 31) is set, dummy2's halves elsewhere
__device__ __forceinline__ uint32_t ev_sel(uint32_t flags, uint32_t addr, uint32_t dummy2)
{
    // sign of byte 1 / byte 3 -> 0xFFFF / 0 per half (PTX prmt sign-replicate
    // mode; the __byte_perm intrinsic masks the selector to 3 bits)
    uint32_t m;
    asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(m) : "r"(flags));
    return (addr & m) | (dummy2 & ~m);
}

constexpr int LINES_NTH = 256;          // 8 warp strips per CTA item
#ifndef LINES_R_DEF
#define LINES_R_DEF 6
#endif
#ifndef LINES_PD_DEF
#define LINES_PD_DEF 2
#endif
constexpr int LINES_R = LINES_R_DEF;    // lattice rows per warp strip
constexpr int LINES_PD = LINES_PD_DEF;  // planes in flight per lane (register ring)
constexpr int LINES_MINUS = 32768;      // byte offset of the minus row (bit 15 of a packed address)

__host__ __device__ inline int lines_nsig(bool fold) { return fold ? 21 : 7; }
__host__ __device__ inline int lines_sig_base(int hs, bool fold)
{
    return (lines_nsig(fold) + 1) * hs <= LINES_MINUS ? hs : LINES_MINUS + hs;
}
__host__ __device__ inline int lines_end(int hs, bool fold)
{
    const int a = LINES_MINUS + hs, b = lines_sig_base(hs, fold) + lines_nsig(fold) * hs;
    return a > b ? a : b;
}

// One warp strip (R lattice rows x 60 lattice columns) marching the planes of
// a chunk [ia, ib).  Shared memory: plus row at 0, minus row at LINES_MINUS
// (EC events of the B/C/D lines, and of the A lines unless FOLD), signature
// rows at sig_base.
template <int DT, int QM, bool VEC, int R, bool FOLD, bool GUARD>
__device__ __forceinline__ void lines_item(const typename Elem<DT>::T* __restrict__ buf, const LGeo& g,
                                           const QuantDev& q, const float* __restrict__ tt, char* __restrict__ h,
                                           int sig_base, int64_t ia, int64_t ib, int j0, int k0, int lane)
{
    using P2 = typename Pair<DT>::T;
    using T = typename Elem<DT>::T;
    constexpr int NR = R + 2;  // cell rows j0-1 .. j0+R held per plane
    constexpr uint32_t FULL = 0xFFFFFFFFu;
    const int Di = (int)g.D;
    const int64_t pe = g.W * g.D;
    const uint32_t sent4 = (uint32_t)(g.M + 1) * 4u;
    const uint32_t hs = (uint32_t)g.hs;
    const float Mf = (float)g.M;
    const int kk = k0 - 2 + 2 * lane;
    const bool computes = lane >= 1 && lane <= 30;
    const uint32_t lmask = computes ? FULL : 0u;  // halo lanes 0 / 31 book nothing
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(h);
    const uint32_t ssig = sb + (uint32_t)sig_base;
    const uint32_t dummy2 = sent4 * 0x10001u;   // sentinel bin of the plus row (never read)
    const int n = (int)(ib - ia);

    // planes t = -1 .. n (plane ia-1+t) exist iff t_lo <= t < t_hi (warp-uniform;
    // only the first two and the last plane of the field can be absent)
    const int t_lo = (int)max((int64_t)-1, 1 - ia);
    const int t_hi = (int)min((int64_t)(n + 2), g.H - ia + 1);
    bool okx = true, oky = true;
    uint32_t rowok = FULL;
    if constexpr (GUARD) {
        okx = kk >= 0 && kk < Di;
        oky = kk >= 0 && kk + 1 < Di;
        rowok = 0;
#pragma unroll
        for (int r = 0; r < NR; ++r) rowok |= (j0 - 1 + r >= 0 && j0 - 1 + r < (int)g.W) ? 1u << r : 0u;
    }
    const uint32_t lanekeep = (okx ? 0x0000FFFFu : 0u) | (oky ? 0xFFFF0000u : 0u);
    // word of row 0 in plane ia-2 (t = -1)
    const T* ptr = buf + ((ia - 2 - g.first) * pe + (int64_t)(j0 - 1) * Di + (okx ? kk : 0));

    auto fetch = [&](int t, const T* at, P2(&dst)[NR]) {
        const bool pin = t >= t_lo && t < t_hi;
        if constexpr (GUARD) {
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                const bool ok = pin && ((rowok >> r) & 1u);
                dst[r] = load_pair<DT, VEC>(at + r * Di, ok && okx, ok && oky);
            }
        } else {
            if (pin) {
#pragma unroll
                for (int r = 0; r < NR; ++r) dst[r] = load_pair<DT, VEC>(at + r * Di, true, true);
            }
        }
    };
    auto quant = [&](int t, const P2(&src)[NR], uint32_t(&V)[NR]) {
        const bool pin = t >= t_lo && t < t_hi;
        if constexpr (GUARD) {
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                const bool ok = pin && ((rowok >> r) & 1u);
                if constexpr (QM == FT_Q_POW2)
                    V[r] = pack_pair_pow2<DT>(src[r], ok ? lanekeep : 0u, q.scale, (uint32_t)g.M * 0x10001u,
                                              sent4 * 0x10001u);
                else
                    V[r] = pack_pair<DT, QM, 0>(src[r], ok && okx, ok && oky, tt, q, g.M, sent4);
            }
        } else if (pin) {
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                if constexpr (QM == FT_Q_POW2)
                    V[r] = pack_pow2_sat<DT>(src[r], q.inv, Mf);
                else
                    V[r] = pack_pair<DT, QM, 0>(src[r], true, true, tt, q, g.M, sent4);
            }
        } else {
#pragma unroll
            for (int r = 0; r < NR; ++r) V[r] = sent4 * 0x10001u;
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

    uint32_t pV[NR], tmi[R + 1], pWm[R + 1], pWp[R + 1];
    uint32_t pB[R + 1], eB[R + 1], pC[R + 1], eC[R + 1], pD[R + 1], eD[R + 1];
    P2 rbuf[LINES_PD][NR];  // planes in flight per lane
    {
        fetch(-1, ptr, rbuf[0]);
        fetch(0, ptr + pe, rbuf[1]);
        uint32_t V0[NR], Wm0[NR], C0[NR], Wm1[NR], C1[NR];
        quant(-1, rbuf[0], V0);  // plane ia-2
        quant(0, rbuf[1], pV);   // plane ia-1
        derive(V0, Wm0, C0);
        derive(pV, Wm1, C1);
#pragma unroll
        for (int r = 1; r <= R; ++r) {
            tmi[r] = hbit(cmp2(V0[r], pV[r]));
            pWm[r] = Wm1[r];
            pWp[r] = shift_pair(pV[r], __shfl_down_sync(FULL, pV[r], 1));
            const uint32_t b0 = vmin2(V0[r - 1], V0[r]), b1 = vmin2(pV[r - 1], pV[r]);
            const uint32_t d0 = vmin2(C0[r - 1], C0[r]), d1 = vmin2(C1[r - 1], C1[r]);
            pB[r] = b1;
            eB[r] = cmp2(b0, b1);
            pC[r] = C1[r];
            eC[r] = cmp2(C0[r], C1[r]);
            pD[r] = d1;
            eD[r] = cmp2(d0, d1);
        }
    }
#pragma unroll
    for (int u = 0; u < LINES_PD; ++u) fetch(1 + u, ptr + (2 + u) * pe, rbuf[u]);
    ptr += (2 + LINES_PD) * pe;  // next fetch: t = 1 + LINES_PD

    // One step: plane t (cell plane p = ia-1+t) arrives in V; every event of
    // cell plane p-1 (whose +i neighbours are now known) is booked.
    auto step = [&](const uint32_t(&V)[NR]) {
        uint32_t Wm[NR], C[NR];
        derive(V, Wm, C);
        uint32_t tpj = 0;
#pragma unroll
        for (int r = 1; r <= R; ++r) {
            const uint32_t W_ = V[r];
            const uint32_t Wp = shift_pair(W_, __shfl_down_sync(FULL, W_, 1));
            // signature of the plane-(p-1) cell: "face neighbour n activates
            // first" = bit 15 / 31 of c' - n + k (k = 0 for -side, -1 for +side)
            const uint32_t cb = pV[r] | 0x80008000u;
            const uint32_t t1 = r == 1 ? hbit(cb - pV[0]) : 0x10001u - tpj;  // -j
            const uint32_t t2 = hbit(cb - pWm[r]);                            // -k
            const uint32_t t3 = hbit(cb - W_ - 0x10001u);                     // +i
            const uint32_t t4 = hbit(cb - pV[r + 1] - 0x10001u);              // +j
            const uint32_t t5 = hbit(cb - pWp[r] - 0x10001u);                 // +k
            uint32_t evS;
            if constexpr (FOLD) {
                // row u + 7 (s_i + 1) = (t1 + t2 + t4 + t5) + 14 - 6 (tmi + t3); no
                // half borrows: 14 - 6 n_i >= 2
                const uint32_t row = (tmi[r] + t3) * (uint32_t)(-6) + (t1 + t2 + t4 + t5 + 0x000E000Eu);
                evS = row * hs + pV[r];
            } else {
                evS = (tmi[r] + t1 + t2 + t3 + t4 + t5) * hs + pV[r];
                // A line event iff both or neither i-neighbour is first; minus (max) iff t3
                const uint32_t fA = ~(tmi[r] ^ t3) & (lmask & 0x00010001u);
                const uint32_t aA = pV[r] | (t3 << 15);
                sinc2(sb, ev_sel(fA << 15, aA, dummy2));
            }
            sinc2(ssig, (evS & lmask) | (dummy2 & ~lmask));  // halo lanes: sentinel bin of row 0
            // B / C / D lines: event iff the along-i order flips at p-1; sign -1
            // (B, C): local min -> minus row; sign +1 (D): local max -> minus row
            const uint32_t B = vmin2(V[r - 1], W_);
            const uint32_t D = vmin2(C[r - 1], C[r]);
            const uint32_t nB = cmp2(pB[r], B), nC = cmp2(pC[r], C[r]), nD = cmp2(pD[r], D);
            sinc2(sb, ev_sel((eB[r] ^ nB) & lmask, pB[r] | (nB & 0x80008000u), dummy2));
            sinc2(sb, ev_sel((eC[r] ^ nC) & lmask, pC[r] | (nC & 0x80008000u), dummy2));
            sinc2(sb, ev_sel((eD[r] ^ nD) & lmask, pD[r] | (~nD & 0x80008000u), dummy2));
            tmi[r] = 0x10001u - t3;
            tpj = t4;
            pWm[r] = Wm[r];
            pWp[r] = Wp;
            pB[r] = B;
            eB[r] = nB;
            pC[r] = C[r];
            eC[r] = nC;
            pD[r] = D;
            eD[r] = nD;
        }
#pragma unroll
        for (int r = 0; r < NR; ++r) pV[r] = V[r];
    };

    // rbuf[u] holds plane t = s + 1 + u at the top of each unrolled round
    uint32_t V[NR];
    for (int s = 0; s < n; s += LINES_PD) {
#pragma unroll
        for (int u = 0; u < LINES_PD; ++u) {
            if (s + u < n) {
                quant(s + u + 1, rbuf[u], V);
                if (s + u + LINES_PD < n) fetch(s + u + 1 + LINES_PD, ptr, rbuf[u]);
                ptr += pe;
                step(V);
            }
        }
    }
}

// GUARD = false: the interior tiles [ti_j0, ti_j1) x [ti_k0, ti_k1), every
// warp strip of which has all its rows and columns inside the field (no load
// predicates, no sentinel selects); GUARD = true: every other tile.  Two
// kernels rather than one branch, so that the boundary code's register
// pressure cannot spill in the interior loop.
template <int DT, int QM, bool VEC, int R, bool FOLD, bool GUARD>
__global__ void __launch_bounds__(LINES_NTH, 2) lines3d_kernel(const typename Elem<DT>::T* __restrict__ buf, LGeo g,
                                                               QuantDev q, unsigned long long* __restrict__ hist)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    char* h = reinterpret_cast<char*>(smem_raw);
    const int M2 = g.M + 2;
    const int hs = g.hs;
    const int sig_base = lines_sig_base(hs, FOLD);
    const int end = lines_end(hs, FOLD);
    float* tt = reinterpret_cast<float*>(h + end);
    for (int i = threadIdx.x; i < end / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(h)[i] = 0;
    if (QM != FT_Q_IDENTITY && QM != FT_Q_POW2)
        for (int i = threadIdx.x; i < M2; i += blockDim.x) tt[i] = q.tt[i];
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x / 32;
    const int nj = g.ti_j1 - g.ti_j0, nk = g.ti_k1 - g.ti_k0;
    const int64_t per_chunk = GUARD ? (int64_t)g.tiles_j * g.tiles_k : (int64_t)nj * nk;
    for (int64_t item = blockIdx.x; item < g.n_items; item += gridDim.x) {
        const int64_t ch = item / per_chunk;
        const int rem = (int)(item - ch * per_chunk);
        int tj, tk;
        if constexpr (GUARD) {
            tj = rem / g.tiles_k;
            tk = rem % g.tiles_k;
            if (tj >= g.ti_j0 && tj < g.ti_j1 && tk >= g.ti_k0 && tk < g.ti_k1) continue;  // the other kernel's
        } else {
            tj = g.ti_j0 + rem / nk;
            tk = g.ti_k0 + rem % nk;
        }
        const int j0 = tj * (8 * R) + warp * R;
        const int k0 = tk * 60;
        const int64_t ia = g.v0 + ch * g.chunk;
        const int64_t ib = min(ia + (int64_t)g.chunk, g.v1);
        lines_item<DT, QM, VEC, R, FOLD, GUARD>(buf, g, q, tt, h, sig_base, ia, ib, j0, k0, lane);
    }
    __syncthreads();
    // fold: C = sum of signature rows, F = sum (6 - u) rows, EC = A events (row
    // groups, or plus/minus when !FOLD) + plus - minus, X = EC - F + C
    const uint32_t* hw = reinterpret_cast<const uint32_t*>(h);
    const int rw = hs / 4, sb = sig_base / 4;
    for (int l = threadIdx.x; l < M2; l += blockDim.x) {
        uint32_t c = 0, f = 0;
        int32_t ec = (int32_t)(hw[l] - hw[LINES_MINUS / 4 + l]);
#pragma unroll
        for (int s = 0; s < lines_nsig(FOLD); ++s) {
            const uint32_t v = hw[sb + s * rw + l];
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

// 16-bit packed signature offsets: (rows - 1) * hs + level * 4 must fit
static bool lines_fold_ok(int M, int hs) { return 20 * hs + (M + 1) * 4 <= 0xFFFF; }
static bool lines_ok(int M)
{
    const int hs = ((M + 2) * 4 + 15) / 16 * 16;
    return (M + 1) * 4 < LINES_MINUS && 6 * hs + (M + 1) * 4 <= 0xFFFF;
}

template <int DT, int QM, bool VEC, bool FOLD, bool GUARD>
static int launch_lines_kernel(const ft_window* win, LGeo g, const QuantDev& qd, size_t smem, int64_t items_per_chunk,
                               int64_t nchunks, uint64_t* hist, cudaStream_t st)
{
    using T = typename Elem<DT>::T;
    if (items_per_chunk <= 0) return FT_OK;
    auto kern = lines3d_kernel<DT, QM, VEC, LINES_R, FOLD, GUARD>;
    FT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    FT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, LINES_NTH, smem));
    if (per_sm < 1) return FT_ERR_ARG;
    g.n_items = (GUARD ? (int64_t)g.tiles_j * g.tiles_k : items_per_chunk) * nchunks;
    const int64_t grid = std::min<int64_t>((int64_t)nsm_l() * per_sm, GUARD ? items_per_chunk * nchunks : g.n_items);
    kern<<<(int)grid, LINES_NTH, smem, st>>>(static_cast<const T*>(win->data), g, qd,
                                            reinterpret_cast<unsigned long long*>(hist));
    FT_CUDA_TRY(cudaGetLastError());
    return FT_OK;
}

template <int DT, int QM, bool VEC, bool FOLD>
static int launch_lines_pair(const ft_window* win, const LGeo& g, const QuantDev& qd, size_t smem, uint64_t* hist,
                             cudaStream_t st)
{
    const int64_t nchunks = cdiv(g.v1 - g.v0, g.chunk);
    const int64_t inner = (int64_t)(g.ti_j1 - g.ti_j0) * (g.ti_k1 - g.ti_k0);
    const int64_t outer = (int64_t)g.tiles_j * g.tiles_k - inner;
    int rc = launch_lines_kernel<DT, QM, VEC, FOLD, false>(win, g, qd, smem, inner, nchunks, hist, st);
    if (rc) return rc;
    return launch_lines_kernel<DT, QM, VEC, FOLD, true>(win, g, qd, smem, outer, nchunks, hist, st);
}

template <int DT, int QM>
static int launch_lines3d(const ft_window* win, int64_t H, int64_t W, int64_t D, int64_t v0, int64_t v1,
                          const ft_quant* qa, int32_t M, uint64_t* hist, cudaStream_t st)
{
    using T = typename Elem<DT>::T;
    constexpr int R = LINES_R, TJ = (LINES_NTH / 32) * R;
    LGeo g{};
    g.H = H; g.W = W; g.D = D; g.v0 = v0; g.v1 = v1; g.first = win->first; g.M = M;
    g.hs = ((M + 2) * 4 + 15) / 16 * 16;
    const bool vec = D % 2 == 0 && reinterpret_cast<uintptr_t>(win->data) % (2 * sizeof(T)) == 0;
    const bool fold = lines_fold_ok(M, g.hs);
    size_t smem = (size_t)lines_end(g.hs, fold);
    if (QM != FT_Q_IDENTITY && QM != FT_Q_POW2) smem += (size_t)(M + 2) * 4;
    g.tiles_j = (int)cdiv(W + 1, TJ);
    g.tiles_k = (int)cdiv(D + 1, 60);
    // interior tiles: every strip's rows j0-1 .. j0+R in [0, W), cells k0-2 .. k0+61 in [0, D)
    g.ti_j0 = 1;
    g.ti_j1 = W >= TJ + 1 ? (int)((W - TJ - 1) / TJ) + 1 : 0;
    g.ti_k0 = 1;
    g.ti_k1 = D >= 62 ? (int)((D - 62) / 60) + 1 : 0;
    if (g.ti_j1 <= g.ti_j0 || g.ti_k1 <= g.ti_k0) g.ti_j0 = g.ti_j1 = g.ti_k0 = g.ti_k1 = 0;
    // plane chunks: enough items to balance ~2 CTAs per SM, marches >= 128 planes
    const int64_t tiles = (int64_t)g.tiles_j * g.tiles_k, rows = v1 - v0;
    int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>(cdiv(16 * 2 * nsm_l(), tiles), rows / 128));
    g.chunk = (int)cdiv(rows, nchunks);
    QuantDev qd = qdev(qa);
    if (QM == FT_Q_POW2) qd.inv = M > 0 ? qd.scale / (float)M : 0.f;
    if (fold)
        return vec ? launch_lines_pair<DT, QM, true, true>(win, g, qd, smem, hist, st)
                   : launch_lines_pair<DT, QM, false, true>(win, g, qd, smem, hist, st);
    return vec ? launch_lines_pair<DT, QM, true, false>(win, g, qd, smem, hist, st)
               : launch_lines_pair<DT, QM, false, false>(win, g, qd, smem, hist, st);
}

}  // namespace ft

#ifndef FT_DEV_KERNEL_ONLY
using namespace ft;

extern "C" int ft_lines3d(const ft_window* win, int64_t H, int64_t W, int64_t D, int64_t v0, int64_t v1,
                          const ft_quant* q, int32_t M, uint64_t* hist, void* stream)
{
    if (!win || !hist || H < 1 || W < 1 || D < 1 || M < 0 || v0 < 0 || v1 > H + 1 || v0 > v1) return FT_ERR_ARG;
    if (W * D > INT32_MAX / 2 || !lines_ok(M)) return FT_ERR_ARG;
    if (v0 == v1) return FT_OK;
    if (!window_ok(win, H, v0, v1, 2)) return FT_ERR_ARG;
    const int qm = effective_qmode(q, true);
    if (qm != FT_Q_IDENTITY && !q->thresholds) return FT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
#ifdef FT_LINES_F32_ONLY  // dev A/B builds (tools/dev/variants.py): the benchmark path only
    if (win->dtype == FT_F32 && qm == FT_Q_POW2)
        return launch_lines3d<FT_F32, FT_Q_POW2>(win, H, W, D, v0, v1, q, M, hist, st);
    return FT_ERR_ARG;
#endif
    switch (win->dtype) {
    case FT_I32:
        if (qm != FT_Q_IDENTITY) return FT_ERR_ARG;
        return launch_lines3d<FT_I32, FT_Q_IDENTITY>(win, H, W, D, v0, v1, q, M, hist, st);
    case FT_U8:
        if (qm == FT_Q_IDENTITY) return launch_lines3d<FT_U8, FT_Q_IDENTITY>(win, H, W, D, v0, v1, q, M, hist, st);
        if (qm == FT_Q_TABLE || qm == FT_Q_POW2)
            return launch_lines3d<FT_U8, FT_Q_TABLE>(win, H, W, D, v0, v1, q, M, hist, st);
        return launch_lines3d<FT_U8, FT_Q_TABLE_ROBUST>(win, H, W, D, v0, v1, q, M, hist, st);
    case FT_U16:
        if (qm == FT_Q_IDENTITY) return launch_lines3d<FT_U16, FT_Q_IDENTITY>(win, H, W, D, v0, v1, q, M, hist, st);
        if (qm == FT_Q_POW2) return launch_lines3d<FT_U16, FT_Q_POW2>(win, H, W, D, v0, v1, q, M, hist, st);
        if (qm == FT_Q_TABLE) return launch_lines3d<FT_U16, FT_Q_TABLE>(win, H, W, D, v0, v1, q, M, hist, st);
        return launch_lines3d<FT_U16, FT_Q_TABLE_ROBUST>(win, H, W, D, v0, v1, q, M, hist, st);
    case FT_F32:
        if (qm == FT_Q_IDENTITY) return FT_ERR_ARG;
        if (qm == FT_Q_POW2) return launch_lines3d<FT_F32, FT_Q_POW2>(win, H, W, D, v0, v1, q, M, hist, st);
        if (qm == FT_Q_TABLE) return launch_lines3d<FT_F32, FT_Q_TABLE>(win, H, W, D, v0, v1, q, M, hist, st);
        return launch_lines3d<FT_F32, FT_Q_TABLE_ROBUST>(win, H, W, D, v0, v1, q, M, hist, st);
    }
    return FT_ERR_ARG;
}

extern "C" int ft_lines3d_ok(int32_t M) { return M >= 0 && lines_ok(M) ? 1 : 0; }
#endif  // FT_DEV_KERNEL_ONLY
