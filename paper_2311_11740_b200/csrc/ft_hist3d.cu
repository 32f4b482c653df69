// ft_hist3d.cu -- 3D vertex-contribution transition histograms (map path).
//
// Replaces the reference's _scan_slabs_3d / _accum_vertex_3d
// (contrib3d.py:241-370).  Per vertex (i, j, k) the eight cells
// (i-1+di, j-1+dj, k-1+dk) are keyed level*8 + slot (slot = di + 2dj + 4dk):
// sorting the keys reproduces the reference's stable insertion argsort
// exactly (ties resolve by slot).  Each sorted rank books ONE event keyed by
// the transition class (type_n -> type_{n+1}, 40 classes)
// instead of the reference's 15 q_in/q_out increments.  The classes of ranks
// 1-3 are a function of the first four sorted slots and those of ranks 4-6 of
// the last four -- and, the pair classes only seeing XORs of slots, of those
// slots RELATIVE to the first / last one: two 512-entry tables (one lookup
// each) classify all six middle ranks; the march kernel keeps a copy per lane
// (or per 4 lanes) in shared memory, the wide kernel reads the 4096-entry
// absolute form from global memory.
//
// Two kernels:
// * hist3d_march (default): a warp marches a strip of vertex rows along i
//   (the slab axis) on packed 16-bit keys, two vertices per word, into a
//   per-CTA shared-memory histogram -- the 41 x (M+2) histogram + tables in
//   shared memory (M <= ~1380);
// * hist3d_wide (any M the reference accepts, e.g. u16 identity levels):
//   one vertex per thread, 32-bit keys, events booked straight into the
//   global u64 histogram.
#include <algorithm>

#include "ft_common.cuh"
#include "ft_lines.cuh"
#include "ft_tables.h"

namespace ft {

constexpr int NTAB = 4096;            // rank-group table entries
constexpr int NXT = 512;              // XOR-relative rank-group table entries
// Classification failures (the reference raises ValueError "3D neighborhood
// outside the configuration table", contrib3d.py:304-305/330, re-raised as
// ClassificationError, contrib3d.py:425-426): table entries of impossible
// slot tuples name the TRAP class; its shared row is never flushed into the
// histogram but sets ft_trap3, which ft_classify_status reports.
constexpr uint32_t TRAP = 40;
constexpr int NROW3 = 41;             // 40 transition classes + the trap row
__device__ unsigned int ft_trap3 = 0;

struct Geo3 {
    int64_t H, W, D, v0, v1, first;
    int M;
    int tiles_j, tiles_k;
    uint32_t c8;  // 8, as a run-time value (Book3)
};

// Class ids of ranks (1,2,3) indexed by the first four sorted slots, and of
// ranks (4,5,6) by the last four (bytes 0..2 of each entry).
struct RankTables {
    uint32_t a[NTAB];
    uint32_t b[NTAB];
    // The pair classes only see XORs of slots (contrib3d.py:76-90), so a rank
    // group's classes are invariant under s -> s ^ c: xa is indexed by the
    // first four sorted slots relative to the first, (s1^s0, s2^s0, s3^s0), xb
    // by the last four relative to the last, (s6^s7, s5^s7, s4^s7) -- 512
    // entries each, small enough to keep one copy PER LANE in shared memory
    // (entry e of lane l at word 32 e + l: bank l, no conflicts).
    uint32_t xa[NXT];
    uint32_t xb[NXT];
};

template <int DT, int QM>
__device__ __forceinline__ uint32_t level3(const typename Elem<DT>::T* __restrict__ buf, const Geo3& g,
                                           int64_t p, int64_t j, int64_t k, const float* tt, const QuantDev& q)
{
    if (p < 0 || p >= g.H || j < 0 || j >= g.W || k < 0 || k >= g.D) return (uint32_t)g.M + 1;
    return to_level<DT, QM>(ld_stream(buf + ((p - g.first) * g.W + j) * g.D + k), tt, q.scale, q.bias,
                            q.negate, g.M);
}

__host__ __device__ __forceinline__ uint32_t slot_index(uint32_t a, uint32_t b, uint32_t c, uint32_t d)
{
    return ((a & 7u) << 9) | ((b & 7u) << 6) | ((c & 7u) << 3) | (d & 7u);
}

// The XOR-relative rank tables, RP copies each (lane l reads copy l % RP:
// entry e at word RP e + l % RP).  RP = 32: one bank per lane, conflict-free;
// RP = 8 (32 KB for both tables) when the histogram leaves no room for more.
template <int RP>
__device__ __forceinline__ void init_shared3(uint32_t* h, uint32_t* ta, uint32_t* tb, float* tt,
                                             const RankTables* __restrict__ rt, const QuantDev& q, int M2,
                                             bool table)
{
    for (int i = threadIdx.x; i < NROW3 * M2; i += blockDim.x) h[i] = 0;
    for (int i = threadIdx.x; i < NXT * RP; i += blockDim.x) {
        ta[i] = rt->xa[i / RP];
        tb[i] = rt->xb[i / RP];
    }
    if (table)
        for (int i = threadIdx.x; i < M2; i += blockDim.x) tt[i] = q.tt[i];
}

__device__ __forceinline__ void flush_hist(const uint32_t* h, unsigned long long* __restrict__ hist, int M2)
{
    for (int i = threadIdx.x; i < 40 * M2; i += blockDim.x) {
        uint32_t v = h[i];
        if (v) atomicAdd(&hist[i], (unsigned long long)v);
    }
    for (int i = threadIdx.x; i < M2; i += blockDim.x)
        if (h[TRAP * M2 + i]) atomicOr(&ft_trap3, 1u);
}

// Two-vertex (packed 16-bit halves) compare-exchange networks: VIMNMX.U16x2.
__device__ __forceinline__ void cswap2(uint32_t& a, uint32_t& b)
{
    const uint32_t lo = __vminu2(a, b);
    b = __vmaxu2(a, b);
    a = lo;
}
__device__ __forceinline__ void sort4x2(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d)
{
    cswap2(a, b);
    cswap2(c, d);
    cswap2(a, c);
    cswap2(b, d);
    cswap2(b, c);
}
__device__ __forceinline__ void merge44x2(uint32_t* k)
{
    cswap2(k[0], k[4]);
    cswap2(k[1], k[5]);
    cswap2(k[2], k[6]);
    cswap2(k[3], k[7]);
    cswap2(k[2], k[4]);
    cswap2(k[3], k[5]);
    cswap2(k[1], k[2]);
    cswap2(k[3], k[4]);
    cswap2(k[5], k[6]);
}

// ------------------------------------------------ register-march map kernel
// A warp marches a strip of HMR vertex rows x 62 vertex columns
// along i; lane l holds the cells (kk, kk+1), kk = k0-1+2l, of HMR+1 cell rows
// as packed level*8 words, so the keys (level*8 + slot) of its two vertices
// share one word and sort4 / merge44 run once per pair (VIMNMX.U16x2); the
// -k cells are one shuffle away.  No staging, no barrier per plane; every
// vertex (j, k) in [0, W] x [0, D] is covered (no edge kernel).
constexpr int HMR = 4;          // vertex rows per warp strip
constexpr int HM3_NTH = 512;    // 16 warps: 64 vertex rows per CTA tile

// Shared-window addresses of the booking step.  Measured on B200 (profiles/
// r02/s5/NOTES.md): the ALU pipe (LOP3 / SHF / LEA / PRMT / VIMNMX, half rate)
// is this kernel's busiest, but IMAD.HI as a right shift is slower than SHF,
// so shifts stay shifts; the class byte of a table entry is selected,
// multiplied by the row stride and added to the level offset by ONE IDP.2A.
struct Book3 {
    uint32_t hb2;      // 2 x shared address of the histogram in both halves: carried by every key
    uint32_t r39;      // 39 S: row 39 is the fixed class of rank 7
    uint32_t ta, tb;   // shared addresses of the lane's copy of the rank tables
    uint32_t S, S16;   // row stride in bytes, 4 (M + 2) (< 2^16), and S << 16
    uint32_t c8;       // 8 as a run-time value: x * c8 + y stays an IMAD
};

// book3 for a packed vertex pair: the rank-group slot indices of both halves
// in one pass, one table lookup per rank group and half, eight increments per
// vertex.  Keys are level * 8 + slot + 2 hb per half (hb = the histogram's
// shared address, a multiple of 4, so order and slot bits are untouched):
// with the slot bits cleared the high half's kc >> 17 -- and the low half's
// (kc << 16) >> 17 -- IS the shared address of the level's bin in row 0.
template <int RP>
__device__ __forceinline__ void book3_pair(const Book3& x, const uint32_t (&k)[8], bool lo, bool hi)
{
    constexpr uint32_t S7 = 0x00070007u, LV = 0xFFF8FFF8u;
    constexpr int SX = RP == 32 ? 9 : 11;  // index in the high half -> table byte offset (* 4 RP)
    // slot indices relative to the first (ranks 1-3) / last (ranks 4-6) sorted slot, 9 bits per half
    const uint32_t a1 = (k[1] ^ k[0]) & S7, a2 = (k[2] ^ k[0]) & S7, a3 = (k[3] ^ k[0]) & S7;
    const uint32_t b1 = (k[6] ^ k[7]) & S7, b2 = (k[5] ^ k[7]) & S7, b3 = (k[4] ^ k[7]) & S7;
    const uint32_t pa = (a1 * x.c8 + a2) * x.c8 + a3;
    const uint32_t pb = (b1 * x.c8 + b2) * x.c8 + b3;
    uint32_t kc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) kc[e] = k[e] & LV;
    auto book = [&](uint32_t ea, uint32_t eb, const uint32_t(&t)[8]) {
        // t[e]: the key of rank e in the HIGH half; class bytes 0..2 of ea / eb
        // select the rows of ranks 1..3 / 4..6 (IDP.2A: S * byte + address)
        ft_sh_inc(t[0] >> 17);
        ft_sh_inc(__dp2a_lo(x.S, ea, t[1] >> 17));
        ft_sh_inc(__dp2a_lo(x.S16, ea, t[2] >> 17));
        ft_sh_inc(__dp2a_hi(x.S, ea, t[3] >> 17));
        ft_sh_inc(__dp2a_lo(x.S, eb, t[4] >> 17));
        ft_sh_inc(__dp2a_lo(x.S16, eb, t[5] >> 17));
        ft_sh_inc(__dp2a_hi(x.S, eb, t[6] >> 17));
        ft_sh_inc((t[7] >> 17) + x.r39);
    };
    if (lo) {
        uint32_t t[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) t[e] = kc[e] << 16;
        book(ft_sh_ld(((pa << 16) >> SX) + x.ta), ft_sh_ld(((pb << 16) >> SX) + x.tb), t);
    }
    if (hi) book(ft_sh_ld((pa >> SX) + x.ta), ft_sh_ld((pb >> SX) + x.tb), kc);
}

template <int DT, int QM, bool VEC, bool EDGE, int RP>
__device__ __forceinline__ void hm3_item(const typename Elem<DT>::T* __restrict__ buf, const Geo3& g,
                                         const QuantDev& q, const float* __restrict__ tt, const Book3& bk,
                                         int64_t ia, int64_t ib, int j0, int k0, int lane)
{
    using P2 = typename Pair<DT>::T;
    using T = typename Elem<DT>::T;
    constexpr int NR = HMR + 1;  // cell rows j0-1 .. j0+HMR-1
    constexpr uint32_t FULL = 0xFFFFFFFFu, K1 = 0x10001u;
    const int Wi = (int)g.W, Di = (int)g.D;
    const uint32_t sent8 = ((uint32_t)g.M + 1u) * 8u;
    const uint32_t S = sent8 * K1 + bk.hb2;  // keys carry 2 hb (book3_pair)
    const int kk = k0 - 1 + 2 * lane;
    const bool clo = lane != 0 && kk >= 0 && kk <= Di, chi = lane != 31 && kk + 1 >= 0 && kk + 1 <= Di;
    const bool okx = kk >= 0 && kk < Di, oky = kk + 1 >= 0 && kk + 1 < Di;
    const int kc = !EDGE ? kk : VEC ? min(max(kk, 0), Di - 2) : min(max(kk, 0), Di - 1);
    uint32_t rowok = (1u << NR) - 1u;
    if constexpr (EDGE) {
        rowok = 0;
#pragma unroll
        for (int c = 0; c < NR; ++c) rowok |= (j0 - 1 + c >= 0 && j0 - 1 + c < Wi) ? 1u << c : 0u;
    }
    bool vrow[HMR];
#pragma unroll
    for (int v = 0; v < HMR; ++v) vrow[v] = j0 + v <= Wi;
    const int64_t pe = g.W * g.D;
    const int n = (int)(ib - ia);
    // planes t = 0 .. n (plane ia-1+t) exist iff t_lo <= t < t_hi
    const int t_lo = (int)max((int64_t)0, 1 - ia);
    const int t_hi = (int)min((int64_t)(n + 1), g.H - ia + 1);
    const T* ptr = buf + ((ia - 1 - g.first) * pe + (int64_t)(j0 - 1) * Di + kc);

    auto fetch = [&](int t, const T* at, P2(&dst)[NR]) {
        if (t >= t_lo && t < t_hi) {
#pragma unroll
            for (int c = 0; c < NR; ++c)
                if (!EDGE || ((rowok >> c) & 1u)) dst[c] = load_pair<DT, VEC>(at + c * Di, true, EDGE ? kk + 1 < Di : true);
        }
    };
    // packed keys (level*8) of one plane's cell rows: V (cells kk, kk+1) and
    // Wm (cells kk-1, kk)
    auto planes = [&](int t, const P2(&src)[NR], uint32_t(&V)[NR], uint32_t(&Wm)[NR]) {
        const bool exists = t >= t_lo && t < t_hi;
#pragma unroll
        for (int c = 0; c < NR; ++c) {
            uint32_t v;
            if constexpr (!EDGE && QM == FT_Q_IDENTITY && (DT == FT_U8 || DT == FT_U16)) {
                v = pack_pair_ident<DT>(src[c], (sent8 >> 3) * K1, 8u, bk.hb2);  // packed clamp + one multiply-add
            } else if constexpr (QM == FT_Q_UMAGIC) {
                // exact integer decoding of u8 / u16 pairs (ft_lines.cuh); absent cells -> sentinel
                v = pack_pair_umagic<DT>(src[c], q, 8u, bk.hb2);
                if constexpr (EDGE) {
                    const uint32_t keep = (okx ? 0x0000FFFFu : 0u) | (oky ? 0xFFFF0000u : 0u);
                    v = (v & keep) | (S & ~keep);
                }
            } else
                v = pack_pair<DT, QM, 1>(src[c], !EDGE || okx, !EDGE || oky, tt, q, g.M, sent8) + bk.hb2;
            if (EDGE && !((rowok >> c) & 1u)) v = S;
            V[c] = exists ? v : S;
            Wm[c] = shift_pair(__shfl_up_sync(FULL, V[c], 1), V[c]);
        }
    };
    // sorted keys of vertex row v from a plane: slots di + 2 dj + 4 dk
    auto keys4 = [&](const uint32_t(&V)[NR], const uint32_t(&Wm)[NR], int v, uint32_t di, uint32_t(&k)[4]) {
        k[0] = Wm[v] + di * K1;
        k[1] = Wm[v + 1] + (2u + di) * K1;
        k[2] = V[v] + (4u + di) * K1;
        k[3] = V[v + 1] + (6u + di) * K1;
        sort4x2(k[0], k[1], k[2], k[3]);
    };

    uint32_t prev[HMR][4];
    P2 ra[NR], rb[NR];
    {
        uint32_t V[NR], Wm[NR];
        fetch(0, ptr, ra);
        planes(0, ra, V, Wm);
#pragma unroll
        for (int v = 0; v < HMR; ++v) keys4(V, Wm, v, 0u, prev[v]);
    }
    fetch(1, ptr + pe, ra);
    fetch(2, ptr + 2 * pe, rb);
    ptr += 3 * pe;  // next fetch: t = 3
    auto step = [&](int t, const P2(&src)[NR]) {
        uint32_t V[NR], Wm[NR];
        planes(t, src, V, Wm);
#pragma unroll
        for (int v = 0; v < HMR; ++v) {
            uint32_t u[4];
            keys4(V, Wm, v, 1u, u);
            uint32_t k8[8] = {prev[v][0], prev[v][1], prev[v][2], prev[v][3], u[0], u[1], u[2], u[3]};
            merge44x2(k8);
            book3_pair<RP>(bk, k8, vrow[v] && clo, vrow[v] && chi);
#pragma unroll
            for (int e = 0; e < 4; ++e) prev[v][e] = u[e] - K1;
        }
    };
    // vertex planes ia + s, s = 0 .. n-1, each reading cell plane t = s+1
    int s = 0;
    for (; s < n; s += 2) {
        step(s + 1, ra);
        if (s + 3 <= n) fetch(s + 3, ptr, ra);
        ptr += pe;
        if (s + 1 >= n) break;
        step(s + 2, rb);
        if (s + 4 <= n) fetch(s + 4, ptr, rb);
        ptr += pe;
    }
}

template <int DT, int QM, bool VEC, int RP>
__global__ void __launch_bounds__(HM3_NTH, 1) hist3d_march(const typename Elem<DT>::T* __restrict__ buf, Geo3 g,
                                                          QuantDev q, const RankTables* __restrict__ rt,
                                                          unsigned long long* __restrict__ hist)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int M2 = g.M + 2;
    uint32_t* h = reinterpret_cast<uint32_t*>(smem_raw);
    uint32_t* ta = h + NROW3 * M2;
    uint32_t* tb = ta + NXT * RP;
    float* tt = reinterpret_cast<float*>(tb + NXT * RP);
    init_shared3<RP>(h, ta, tb, tt, rt, q, M2, QM != FT_Q_IDENTITY && QM != FT_Q_POW2 && QM != FT_Q_UMAGIC);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Book3 bk;
    // 16-bit keys: level * 8 + slot + 2 hb (hb = 0x400 on B200; the launcher
    // keeps M + 1 <= 4095, so hb up to ~16 KB would still fit)
    const uint32_t hb = (uint32_t)__cvta_generic_to_shared(h);
    if (2u * hb + 8u * (uint32_t)M2 > 0xFFFFu) __trap();
    bk.hb2 = 2u * hb * 0x10001u;
    bk.S = 4u * (uint32_t)M2;
    bk.S16 = bk.S << 16;
    bk.r39 = 39u * bk.S;
    bk.ta = (uint32_t)__cvta_generic_to_shared(ta) + 4u * (lane % RP);
    bk.tb = (uint32_t)__cvta_generic_to_shared(tb) + 4u * (lane % RP);
    bk.c8 = g.c8;
    constexpr int TJ = (HM3_NTH / 32) * HMR;
    const int64_t np = g.v1 - g.v0;
    const int64_t T = (int64_t)g.tiles_j * g.tiles_k * np;  // (tile, plane) units, tile-major
    const int64_t u_end = T * (blockIdx.x + 1) / gridDim.x;
    for (int64_t u = T * blockIdx.x / gridDim.x; u < u_end;) {
        const int tile = (int)(u / np);
        const int64_t p = u - (int64_t)tile * np;
        const int64_t len = min(u_end - u, np - p);
        u += len;
        const int tj = tile / g.tiles_k;
        const int j0 = tj * TJ + warp * HMR;
        const int k0 = (tile - tj * g.tiles_k) * 62 - 1;
        if (j0 > g.W) continue;
        const int64_t ia = g.v0 + p;
        if (j0 >= 1 && j0 + HMR <= g.W && k0 >= 1 && k0 + 63 <= g.D)
            hm3_item<DT, QM, VEC, false, RP>(buf, g, q, tt, bk, ia, ia + len, j0, k0, lane);
        else
            hm3_item<DT, QM, VEC, true, RP>(buf, g, q, tt, bk, ia, ia + len, j0, k0, lane);
    }
    __syncthreads();
    flush_hist(h, hist, M2);
}

// Any level count: one vertex per thread (k fastest: coalesced cell loads,
// the 8 neighbours of a vertex hit L1), 32-bit keys level*8 + slot, the
// 8 events booked straight into the global u64 histogram (L2 atomics).  The
// threshold table of a quantized input is read from global memory.
template <int DT, int QM>
__global__ void __launch_bounds__(256) hist3d_wide(const typename Elem<DT>::T* __restrict__ buf, Geo3 g,
                                                   QuantDev q, const RankTables* __restrict__ rt,
                                                   unsigned long long* __restrict__ hist)
{
    const uint64_t M2 = (uint64_t)g.M + 2;
    const int64_t nj = g.W + 1, nk = g.D + 1;
    const int64_t n = (g.v1 - g.v0) * nj * nk;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t % nk;
        const int64_t r = t / nk;
        const int64_t j = r % nj;
        const int64_t i = g.v0 + r / nj;
        uint32_t a[8];
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            // slot s = di + 2 dj + 4 dk (contrib3d.py:47-49); sorted in two
            // groups of four (dk = 0 / 1) and merged
            const int di = s & 1, dj = (s >> 1) & 1, dk = s >> 2;
            a[(s & 3) + 4 * dk] = level3<DT, QM>(buf, g, i - 1 + di, j - 1 + dj, k - 1 + dk, q.tt, q) * 8u + s;
        }
        sort4(a[0], a[1], a[2], a[3]);
        sort4(a[4], a[5], a[6], a[7]);
        merge44(a);
        const uint32_t ea = rt->a[slot_index(a[0], a[1], a[2], a[3])];
        const uint32_t eb = rt->b[slot_index(a[4], a[5], a[6], a[7])];
        const uint32_t cls[8] = {0u, ea & 0xFFu, (ea >> 8) & 0xFFu, ea >> 16, eb & 0xFFu, (eb >> 8) & 0xFFu,
                                 eb >> 16, 39u};
#pragma unroll
        for (int r8 = 0; r8 < 8; ++r8) {
            if (cls[r8] < TRAP)
                atomicAdd(&hist[cls[r8] * M2 + (a[r8] >> 3)], 1ull);
            else
                atomicOr(&ft_trap3, 1u);
        }
    }
}

// Rank-group tables from the step table: simulate the active-slot masks of
// every ordered slot 4-tuple.
static RankTables make_rank_tables()
{
    const Tables& t = tables(3);
    RankTables rt{};
    for (int idx = 0; idx < NTAB; ++idx) {
        const int s[4] = {idx >> 9 & 7, idx >> 6 & 7, idx >> 3 & 7, idx & 7};
        bool distinct = true;
        for (int x = 0; x < 4; ++x)
            for (int y = x + 1; y < 4; ++y) distinct &= s[x] != s[y];
        rt.a[idx] = rt.b[idx] = TRAP * 0x010101u;
        if (!distinct) continue;  // unreachable: a vertex's 8 slots are distinct
        // ranks 1..3: masks {s0}, {s0,s1}, {s0,s1,s2}
        int m = 1 << s[0];
        uint32_t ea = 0;
        for (int r = 1; r <= 3; ++r) {
            const int c = t.step[m * 8 + s[r]];
            ea |= (uint32_t)(c >= 0 ? c : (int)TRAP) << (8 * (r - 1));
            m |= 1 << s[r];
        }
        rt.a[idx] = ea;
        // ranks 4..6 given sorted slots s4..s7 = s[0..3]: before rank 4 the
        // active set is the complement of {s4..s7}
        int mb = 0xFF & ~((1 << s[0]) | (1 << s[1]) | (1 << s[2]) | (1 << s[3]));
        uint32_t eb = 0;
        for (int r = 0; r < 3; ++r) {
            const int c = t.step[mb * 8 + s[r]];
            eb |= (uint32_t)(c >= 0 ? c : (int)TRAP) << (8 * r);
            mb |= 1 << s[r];
        }
        rt.b[idx] = eb;
    }
    // XOR-relative tables; an entry whose class triple is NOT the same for
    // every base slot (cannot happen: the pair classes only see XORs) is left
    // as the trap class, so a broken invariance would fail loudly.
    for (int idx = 0; idx < NXT; ++idx) {
        const int x1 = idx >> 6 & 7, x2 = idx >> 3 & 7, x3 = idx & 7;
        rt.xa[idx] = rt.xb[idx] = TRAP * 0x010101u;
        if (!x1 || !x2 || !x3 || x1 == x2 || x1 == x3 || x2 == x3) continue;
        const uint32_t ea = rt.a[slot_index(0, x1, x2, x3)], eb = rt.b[slot_index(x3, x2, x1, 0)];
        bool same = true;
        for (int c = 1; c < 8; ++c)
            same &= rt.a[slot_index(c, x1 ^ c, x2 ^ c, x3 ^ c)] == ea && rt.b[slot_index(x3 ^ c, x2 ^ c, x1 ^ c, c)] == eb;
        if (same) {
            rt.xa[idx] = ea;
            rt.xb[idx] = eb;
        }
    }
    return rt;
}

static int sm_count()
{
    int dev = 0, n = kSMs;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

// Per-device copy of the rank tables (uploaded once).
static const RankTables* device_rank_tables()
{
    static const RankTables host = make_rank_tables();
    static RankTables* dev_tabs[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    if (!dev_tabs[dev]) {
        RankTables* p = nullptr;
        if (cudaMalloc(&p, sizeof(RankTables)) != cudaSuccess) return nullptr;
        if (cudaMemcpy(p, &host, sizeof(RankTables), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
        dev_tabs[dev] = p;
    }
    return dev_tabs[dev];
}

// shared bytes of hist3d_march: the 41 x (M+2) histogram, RP copies of both rank tables, the threshold table
static size_t march3_smem(int M, int rp) { return (size_t)(NROW3 * (M + 2) + 2 * NXT * rp + (M + 2)) * 4; }
static bool march3_ok(int M) { return M + 1 <= 4095 && march3_smem(M, 8) <= 227 * 1024; }
// one table copy per lane (128 KB) beside the histogram: M <= 601
static bool march3_rp32(int M) { return march3_smem(M, 32) <= 227 * 1024; }

template <int DT, int QM>
static int launch3(const ft_window* win, int64_t H, int64_t W, int64_t D, int64_t v0, int64_t v1,
                   const ft_quant* qa, int32_t M, uint64_t* hist, cudaStream_t st)
{
    using T = typename Elem<DT>::T;
    const RankTables* rt = device_rank_tables();
    if (!rt) return FT_ERR_CUDA_BASE + (int)cudaErrorMemoryAllocation;
    const T* buf = static_cast<const T*>(win->data);
    Geo3 g{};
    g.H = H; g.W = W; g.D = D; g.v0 = v0; g.v1 = v1; g.first = win->first; g.M = M;
    QuantDev q{qa ? qa->mode : FT_Q_IDENTITY, qa ? qa->negate : 0, qa ? qa->scale : 0.f, qa ? qa->bias : 0.f,
               qa ? qa->thresholds : nullptr};
    if (QM == FT_Q_UMAGIC && !umagic_fill(qa, M, DT == FT_U8 ? 256 : 65536, q)) return FT_ERR_INTERNAL;
    auto* out = reinterpret_cast<unsigned long long*>(hist);
    const int nsm = sm_count();
    if (march3_ok(M)) {
        // register march: every vertex (j, k) in [0, W] x [0, D]
        const bool wide = march3_rp32(M);
        const size_t sm = march3_smem(M, wide ? 32 : 8);
        const bool vec = D % 2 == 0 && reinterpret_cast<uintptr_t>(buf) % (2 * sizeof(T)) == 0;
        auto kern = wide ? (vec ? hist3d_march<DT, QM, true, 32> : hist3d_march<DT, QM, false, 32>)
                         : (vec ? hist3d_march<DT, QM, true, 8> : hist3d_march<DT, QM, false, 8>);
        g.c8 = 8;
        FT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        int per_sm = 0;
        FT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, HM3_NTH, sm));
        if (per_sm < 1) return FT_ERR_INTERNAL;
        g.tiles_j = (int)cdiv(W + 1, (HM3_NTH / 32) * HMR);
        g.tiles_k = (int)((D + 1) / 62 + 1);  // tile t: vertex columns 62 t - 1 .. 62 t + 60
        const int64_t work = (int64_t)g.tiles_j * g.tiles_k * (v1 - v0);
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)nsm * per_sm, cdiv(work, 32)));
        kern<<<grid, HM3_NTH, sm, st>>>(buf, g, q, rt, out);
        FT_CUDA_TRY(cudaGetLastError());
        return FT_OK;
    }
    const int64_t n = (v1 - v0) * (W + 1) * (D + 1);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), (int64_t)nsm * 8));
    constexpr int QW = QM == FT_Q_POW2 || QM == FT_Q_UMAGIC ? FT_Q_TABLE : QM;  // the table ships with these too
    hist3d_wide<DT, QW><<<grid, 256, 0, st>>>(buf, g, q, rt, out);
    FT_CUDA_TRY(cudaGetLastError());
    return FT_OK;
}

}  // namespace ft

using namespace ft;

extern "C" int ft_classify_status(void* stream)
{
    FT_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    unsigned int v = 0;
    FT_CUDA_TRY(cudaMemcpyFromSymbol(&v, ft_trap3, sizeof(v)));
    if (v) {
        const unsigned int zero = 0;
        FT_CUDA_TRY(cudaMemcpyToSymbol(ft_trap3, &zero, sizeof(zero)));
    }
    return v ? FT_ERR_CLASSIFY : FT_OK;
}

extern "C" int ft_debug_trap_tables(int32_t on)
{
    const RankTables* d = device_rank_tables();
    if (!d) return FT_ERR_CUDA_BASE + (int)cudaErrorMemoryAllocation;
    static const RankTables good = make_rank_tables();
    static const RankTables bad = [] {
        RankTables r = make_rank_tables();
        for (int i = 0; i < NTAB; ++i) r.a[i] = r.b[i] = TRAP * 0x010101u;
        for (int i = 0; i < NXT; ++i) r.xa[i] = r.xb[i] = TRAP * 0x010101u;
        return r;
    }();
    FT_CUDA_TRY(cudaMemcpy(const_cast<RankTables*>(d), on ? &bad : &good, sizeof(RankTables), cudaMemcpyHostToDevice));
    return FT_OK;
}

extern "C" int ft_hist3d(const ft_window* win, int64_t H, int64_t W, int64_t D, int64_t v0, int64_t v1,
                         const ft_quant* q, int32_t M, uint64_t* hist, void* stream)
{
    if (!win || !hist || H < 1 || W < 1 || D < 1 || M < 0 || v0 < 0 || v1 > H + 1 || v0 > v1) return FT_ERR_ARG;
    if (W * D > INT32_MAX / 2) return FT_ERR_ARG;  // 32-bit in-plane offsets
    if (v0 == v1) return FT_OK;
    // every plane a vertex row in [v0, v1) reads must be resident
    const int64_t need_lo = std::max<int64_t>(v0 - 1, 0), need_hi = std::min<int64_t>(v1 - 1, H - 1);
    if (need_lo <= need_hi && (win->data == nullptr || need_lo < win->first || need_hi >= win->first + win->count))
        return FT_ERR_ARG;
    if (M > (1 << 28) - 2) return FT_ERR_ARG;  // keys level*8 + slot in 32 bits
    // FT_Q_POW2 (lo = 0, hi = 2^p): the march quantizes without the table
    const int qm = effective_qmode(q, true);
    if (qm != FT_Q_IDENTITY && (!q->thresholds || win->dtype == FT_I32)) return FT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    QuantDev probe{};
    switch (win->dtype) {
    case FT_I32:
        if (qm != FT_Q_IDENTITY) return FT_ERR_ARG;
        return launch3<FT_I32, FT_Q_IDENTITY>(win, H, W, D, v0, v1, q, M, hist, st);
    case FT_U8:
        if (qm == FT_Q_IDENTITY) return launch3<FT_U8, FT_Q_IDENTITY>(win, H, W, D, v0, v1, q, M, hist, st);
        if (march3_ok(M) && umagic_fill(q, M, 256, probe)) return launch3<FT_U8, FT_Q_UMAGIC>(win, H, W, D, v0, v1, q, M, hist, st);
        if (qm == FT_Q_TABLE || qm == FT_Q_POW2) return launch3<FT_U8, FT_Q_TABLE>(win, H, W, D, v0, v1, q, M, hist, st);
        return launch3<FT_U8, FT_Q_TABLE_ROBUST>(win, H, W, D, v0, v1, q, M, hist, st);
    case FT_U16:
        if (qm == FT_Q_IDENTITY) return launch3<FT_U16, FT_Q_IDENTITY>(win, H, W, D, v0, v1, q, M, hist, st);
        // integer ranges (the data's min / max): exact integer decoding in the march kernel, no table
        if (march3_ok(M) && umagic_fill(q, M, 65536, probe)) return launch3<FT_U16, FT_Q_UMAGIC>(win, H, W, D, v0, v1, q, M, hist, st);
        if (qm == FT_Q_POW2) return launch3<FT_U16, FT_Q_POW2>(win, H, W, D, v0, v1, q, M, hist, st);
        if (qm == FT_Q_TABLE) return launch3<FT_U16, FT_Q_TABLE>(win, H, W, D, v0, v1, q, M, hist, st);
        return launch3<FT_U16, FT_Q_TABLE_ROBUST>(win, H, W, D, v0, v1, q, M, hist, st);
    case FT_F32:
        if (qm == FT_Q_IDENTITY) return FT_ERR_ARG;
        if (qm == FT_Q_POW2) return launch3<FT_F32, FT_Q_POW2>(win, H, W, D, v0, v1, q, M, hist, st);
        if (qm == FT_Q_TABLE) return launch3<FT_F32, FT_Q_TABLE>(win, H, W, D, v0, v1, q, M, hist, st);
        return launch3<FT_F32, FT_Q_TABLE_ROBUST>(win, H, W, D, v0, v1, q, M, hist, st);
    }
    return FT_ERR_ARG;
}
