// unpack.cuh — the 2-bit -> int8 level expansion used by every tensor-core path.
//
// The paper's unpack step (§3.1, Alg. 1 line 9: mask/shift the packed codes) produces
// here the int8 LEVEL of each code instead of a LUT index: one PRMT (byte permute) looks up 4
// codes at once in the 4-byte level table L = {l[0], l[1], l[2], l[3]} (the product
// table is wl (x) al, so T[(w<<2)|a] = wl[w]*al[a] is one int8 MMA term).
//
// Byte order: the 16 codes of a 32-bit word come out as
//     0,2,4,6, 8,10,12,14, 1,3,5,7, 9,11,13,15
// Both GEMM operands are expanded with this same function, so the permutation is common to
// the two K axes and the dot product is unchanged.
#pragma once
#include <stdint.h>

namespace dg {

__device__ __forceinline__ uint32_t prmt_b32(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

// 16 packed codes (code k at bits 2k) -> 4 words of int8 levels in the order above.
__device__ __forceinline__ uint4 unpack16_levels(uint32_t x, uint32_t L) {
    const uint32_t X = x & 0x33333333u, Y = (x >> 2) & 0x33333333u;
    return make_uint4(prmt_b32(L, L, X), prmt_b32(L, L, X >> 16), prmt_b32(L, L, Y), prmt_b32(L, L, Y >> 16));
}

inline uint32_t pack_levels_i8(const int32_t l[4]) {
    uint32_t L = 0;
    for (int i = 0; i < 4; ++i) L |= ((uint32_t)(l[i] & 0xFF)) << (8 * i);
    return L;
}

}  // namespace dg
