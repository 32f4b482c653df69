// ft_lines.cuh -- device helpers shared by the line-decomposition curve
// kernels (ft_lines.cu: 3D, ft_lines2d.cu: 2D): packed 16-bit bin offsets, the
// FMA-pipe quantizer, the dummy-address shared increments, the shared layout.
#pragma once
#include <algorithm>
#include <cmath>
#include <mutex>

#include "ft_lattice.cuh"

namespace ft {

// Packed level words hold, per 16-bit half, the bin's offset BELOW the top of
// its histogram region: rel = row * hs + (level + 1) * 4 (rel = 0 is the
// region's dummy word).  The regions are laid out downward (lines_layout), so
// the shared address of a bin is top - rel and ONE IDP.2A per half does the
// half split, the event select and the address:
//     addr = top + h0 * b0 + h1 * b1,   (b0, b1) signed bytes, -1 or 0
// -- a half whose flag byte is 0 lands on the dummy word at top (sinc2).
constexpr uint32_t LINES_REL0 = 0x00040004u;  // rel of level 0 in row 0, both halves
// bit 15 / 31 of x as 0 / 255 in each 16-bit half: ONE PRMT (sign-replicate
// byte 1 / byte 3 into byte 0 / byte 2, zero bytes 1 / 3) instead of a shift
// and a mask -- the signature counts run in units of 255 (row stride 255 K).
__device__ __forceinline__ uint32_t hff(uint32_t x)
{
    uint32_t m;
    asm("prmt.b32 %0, %1, 0, 0x4B49;" : "=r"(m) : "r"(x));
    return m;
}
constexpr uint32_t FF2 = 0x00FF00FFu;  // 255 in both halves
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
__device__ __forceinline__ uint32_t pack_pow2_sat(const typename Pair<DT>::T& v, float inv, float Mf, uint32_t four,
                                                  uint32_t sb2)
{
    const float a = __saturatef((float)v.x * inv);
    const float b = __saturatef((float)v.y * inv);
    // both cells at once: FFMA2.RM then FADD2.RM (packed f32x2, sm_100)
    const unsigned long long ab = ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(a);
    const unsigned long long m2 = ((unsigned long long)__float_as_uint(Mf) << 32) | __float_as_uint(Mf);
    unsigned long long y, z;
    asm("fma.rm.f32x2 %0, %1, %2, %3;" : "=l"(y) : "l"(ab), "l"(m2), "l"(0x3F0000003F000000ull));
    asm("add.rm.f32x2 %0, %1, %2;" : "=l"(z) : "l"(y), "l"(0x4B0000004B000000ull));
    return __byte_perm((uint32_t)z, (uint32_t)(z >> 32), 0x5410) * four + sb2;  // IMAD: FMA pipe
}

// FT_Q_UMAGIC: uint8 / uint16 pairs decoded in exact integer arithmetic.  For
// integers x, lo < hi the reference level clip(floor((x - lo) M / (hi - lo) +
// 0.5), 0, M) (fields.py:20-33) is floor((2 t M + R) / (2 R)) with t =
// clamp(x, lo, hi) - lo and R = hi - lo: the numerator stays below 2^31 and
// the division by 2 R is a multiply-high and a shift (Granlund-Montgomery),
// all of it checked against the float64 formula for EVERY input value on the
// host before a range is used (umagic_fill).  Two packed clamps, no
// int<->float conversion (the quarter-rate XU pipe), no table load.
template <int DT>
__device__ __forceinline__ uint32_t pack_pair_umagic(const typename Pair<DT>::T& v, const QuantDev& q, uint32_t four,
                                                     uint32_t rel0)
{
    uint32_t w;
    if constexpr (DT == FT_U16)
        w = *reinterpret_cast<const uint32_t*>(&v);  // a ushort2 IS the packed word
    else
        w = __byte_perm((uint32_t)v.x, (uint32_t)v.y, 0x5410);
    const uint32_t t2 = __vmaxu2(__vminu2(w, q.u_hi2), q.u_lo2) - q.u_lo2;
    const uint32_t l0 = __umulhi((t2 & 0xFFFFu) * q.u_mul + q.u_add, q.u_magic) >> q.u_shift;
    const uint32_t l1 = __umulhi((t2 >> 16) * q.u_mul + q.u_add, q.u_magic) >> q.u_shift;
    return l1 * (four << 16) + (l0 * four + rel0);  // two IMADs (FMA pipe) instead of a PRMT + IMAD
}

// Identity levels of uint8 / uint16 pairs (C3: u8 images), packed: the pair as
// two 16-bit halves (u8: one PRMT; u16: the loaded word), one packed min with
// the sentinel M + 1 (the scalar path's clamp, ft_common.cuh to_level) and one
// IMAD -- instead of a convert / min / shift per cell and a PRMT.
template <int DT>
__device__ __forceinline__ uint32_t pack_pair_ident(const typename Pair<DT>::T& v, uint32_t sent_lv2, uint32_t four,
                                                    uint32_t rel0)
{
    uint32_t w;
    if constexpr (DT == FT_U16) {
        w = *reinterpret_cast<const uint32_t*>(&v);
    } else {
        static_assert(DT == FT_U8, "packed identity levels: uint8 / uint16 only");
        w = __byte_perm((uint32_t)*reinterpret_cast<const uint16_t*>(&v), 0u, 0x4140);
    }
    return __vminu2(w, sent_lv2) * four + rel0;
}

// Host side of FT_Q_UMAGIC: true (and qd filled) iff the input type has nvals
// = 256 / 65536 values, the range is an increasing integer one inside it and
// the integer formula reproduces the float64 reference for every value.
static inline bool umagic_fill(const ft_quant* qa, int M, int nvals, QuantDev& qd)
{
    if (!qa || qa->negate || M < 1 || !(qa->lo < qa->hi)) return false;
    if (qa->mode != FT_Q_TABLE && qa->mode != FT_Q_TABLE_ROBUST && qa->mode != FT_Q_POW2) return false;
    const double lo = qa->lo, hi = qa->hi;
    if (lo < 0 || hi > nvals - 1 || lo != (double)(int64_t)lo || hi != (double)(int64_t)hi) return false;
    const uint64_t L = (uint64_t)lo, R = (uint64_t)hi - L, mul = 2ull * (uint64_t)M, d = 2 * R;
    if (R * mul + R >= (1ull << 31)) return false;
    int lg = 0;
    while ((1ull << lg) < d) ++lg;  // ceil(log2 d) >= 1
    const uint64_t magic = ((1ull << (31 + lg)) + d - 1) / d;
    if (magic >> 32) return false;
    // one verified range is remembered (the usual case: one field, many launches)
    static std::mutex mu;
    static double c_lo = 0, c_hi = 0;
    static int c_M = 0, c_n = 0;
    std::lock_guard<std::mutex> lock(mu);
    if (!(c_lo == lo && c_hi == hi && c_M == M && c_n == nvals)) {
        for (int x = 0; x < nvals; ++x) {
            const uint64_t t = (uint64_t)std::min<int64_t>(std::max<int64_t>(x, (int64_t)L), (int64_t)(L + R)) - L;
            const uint64_t lev = ((t * mul + R) * magic) >> (31 + lg);
            const double ref = std::min(std::max(std::floor(((double)x - lo) * (double)M / (hi - lo) + 0.5), 0.0), (double)M);
            if ((double)lev != ref) return false;
        }
        c_lo = lo; c_hi = hi; c_M = M; c_n = nvals;
    }
    qd.u_lo2 = (uint32_t)L * 0x10001u;
    qd.u_hi2 = (uint32_t)(L + R) * 0x10001u;
    qd.u_mul = (uint32_t)mul;
    qd.u_add = (uint32_t)R;
    qd.u_magic = (uint32_t)magic;
    qd.u_shift = (uint32_t)(lg - 1);
    return true;
}

// Shared-memory increments of both 16-bit halves of a packed word of bin
// offsets.  No predicates (ptxas turns predicated shared atomics into
// branches): sel holds a flag byte per half, byte 0 for the low half and byte
// 3 for the high one (0xFF = book the bin, 0 = no event: the dummy word at
// top; all such lanes hit the same word, one bank access merged by the POPC
// increment), bytes 1 and 2 zero.  The two IDP.2A run on the FMA pipe, the ALU
// pipe being the busy one; an earlier IMAD.HI + IMAD split cost 4.4 % of the
// C5 kernel (IMAD.HI is a slow instruction on B200; profiles/r02/s5/NOTES.md).
__device__ __forceinline__ void sinc2(uint32_t rel2, uint32_t sel, uint32_t top)
{
    uint32_t lo, hi;
    asm("dp2a.lo.u32.s32 %0, %1, %2, %3;" : "=r"(lo) : "r"(rel2), "r"(sel), "r"(top));
    asm("dp2a.hi.u32.s32 %0, %1, %2, %3;" : "=r"(hi) : "r"(rel2), "r"(sel), "r"(top));
    ft_check_smem(lo);
    ft_check_smem(hi);
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(lo));
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(hi));
}
// sinc2 selector of a lane's dense event: every half it computes (lane 0 only
// its high half, lane 31 only its low one: the others are the halo cells)
__device__ __forceinline__ uint32_t lane_sel(int lane)
{
    return lane == 0 ? 0xFF000000u : lane == 31 ? 0x000000FFu : 0xFF0000FFu;
}
// sinc2 selector from event flags in bits 15 / 31: ONE PRMT (sign-replicate
// byte 1 into byte 0 and byte 3 into byte 3, zero bytes 1 and 2)
__device__ __forceinline__ uint32_t ev_sel(uint32_t flags)
{
    uint32_t m;
    asm("prmt.b32 %0, %1, 0, 0xB449;" : "=r"(m) : "r"(flags));
    return m;
}
// (a & m) | (b & ~m) as ONE LOP3 (left to itself ptxas sometimes splits it
// into two around a hoisted b & ~m)
__device__ __forceinline__ uint32_t sel_mask(uint32_t m, uint32_t a, uint32_t b)
{
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(d) : "r"(m), "r"(a), "r"(b));
    return d;
}
// Shared layout of the line kernels (byte offsets from the dynamic block),
// every region growing DOWNWARD from its top:
//   signature bins (row s, level l) at dtop - (s hs + (l + 1) 4), the dense
//     dummy word at dtop;
//   minus-row bins at ptop - 32768 - (l + 1) 4 (bit 15 of a sparse offset
//     selects the minus row), just above dtop;
//   plus-row bins at ptop - (l + 1) 4, the sparse dummy word at ptop;
//   the threshold table in the gap above the minus row.
// 16-bit halves: (nsig - 1) hs + (M + 2) 4 < 65536 and 2 (M + 2) 4 <= 32768.
constexpr int LINES_MINUS = 32768;
struct LLay {
    int dtop, ptop, tt, end;
};
__host__ __device__ inline LLay lines_layout(int hs, int nsig, int M)
{
    const int m4 = (M + 2) * 4;
    LLay L;
    L.dtop = ((nsig - 1) * hs + m4 + 15) & ~15;
    L.ptop = (L.dtop + 16 + LINES_MINUS + m4 + 15) & ~15;
    L.tt = L.ptop - LINES_MINUS;
    L.end = L.ptop + 16;
    return L;
}
__host__ __device__ inline bool lines_layout_ok(int hs, int nsig, int M)
{
    const int m4 = (M + 2) * 4;
    return m4 <= hs && (nsig - 1) * hs + m4 < 65536 && 2 * m4 <= LINES_MINUS;
}

}  // namespace ft
