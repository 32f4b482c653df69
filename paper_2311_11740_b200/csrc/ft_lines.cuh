// ft_lines.cuh -- device helpers shared by the line-decomposition curve
// kernels (ft_lines.cu: 3D, ft_lines2d.cu: 2D): packed 16-bit level words that
// carry the shared base of the histogram block, the FMA-pipe quantizer, the
// dummy-address shared increments.
#pragma once
#include "ft_lattice.cuh"

namespace ft {

// Packed level words carry the shared-space address of the kernel's dynamic
// shared block in both halves (sb2 = base * 0x10001), read at run time with
// cvta (lines_sb2); the host-side fit checks use the base the probe kernel
// measured once per process (lines_sbase: 0x400 on B200, the 1 KB the
// hardware reserves).
constexpr uint32_t LINES_SBASE_DEFAULT = 0x400;
__device__ __forceinline__ uint32_t lines_sb2(const void* smem)
{
    return (uint32_t)__cvta_generic_to_shared(smem) * 0x10001u;
}

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

// Shared-memory increments of both 16-bit halves of a packed address.  No
// predicates: ptxas turns predicated shared atomics into branches, so a lane
// without an event points at a DUMMY word instead (all such lanes hit the
// same word: one bank access, merged by the POPC increment).  The halves are
// split on the FMA pipe, the ALU pipe being the busy one, by two IDP.2A
// (addr.h0 * b0 + addr.h1 * b1 with (b0, b1) = (1, 0) / (0, 1)): the earlier
// IMAD.HI / IMAD pair cost 4.4 % of the C5 kernel (IMAD.HI is a slow
// instruction on B200; profiles/r02/s5/NOTES.md).
// Packed level words carry the shared address of the block (sb2, in every
// half), so a half IS the shared address of a signature bin and the
// plus/minus rows are an immediate above it: ATOMS [R + imm], no base add.
template <int OFF>
__device__ __forceinline__ void sinc2(uint32_t addr)
{
    const uint32_t hi = __dp2a_lo(addr, 0x0100u, 0u);
    const uint32_t lo = __dp2a_lo(addr, 0x0001u, 0u);
    ft_check_smem(lo + OFF);
    ft_check_smem(hi + OFF);
    asm volatile("red.shared.add.u32 [%0+%1], 1;" ::"r"(lo), "n"(OFF));
    asm volatile("red.shared.add.u32 [%0+%1], 1;" ::"r"(hi), "n"(OFF));
}
// (a & m) | (b & ~m) as ONE LOP3 (left to itself ptxas sometimes splits it
// into two around a hoisted b & ~m)
__device__ __forceinline__ uint32_t sel_mask(uint32_t m, uint32_t a, uint32_t b)
{
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xCA;" : "=r"(d) : "r"(m), "r"(a), "r"(b));
    return d;
}
// halves of addr whose flag bit (15 / 31) is set, dummy2's halves elsewhere
__device__ __forceinline__ uint32_t ev_sel(uint32_t flags, uint32_t addr, uint32_t dummy2)
{
    // sign of byte 1 / byte 3 -> 0xFFFF / 0 per half (PTX prmt sign-replicate
    // mode; the __byte_perm intrinsic masks the selector to 3 bits)
    uint32_t m;
    asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(m) : "r"(flags));
    return sel_mask(m, addr, dummy2);
}

// Shared layout of the line kernels: signature rows at 0 (at most 64 KB: the
// 16-bit packed row offsets), the plus row at LINES_PLUS and the minus row
// LINES_MINUS above it; both are constants, so every ATOMS address is
// [R + imm].
constexpr int LINES_MINUS = 32768;      // byte offset of the minus row (bit 15 of a packed address)
constexpr int LINES_PLUS = 65536;

// Probes once per process where dynamic shared memory starts (the kernels
// address it absolutely and the 16-bit packed offsets must fit below 64 KB):
// FT_OK or an error code; lines_sbase() is the measured base (the default
// until the probe ran).
int lines_check_sbase();
int lines_sbase();

}  // namespace ft
