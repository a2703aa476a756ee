// requant16.cuh — the 16-bit SIMD requantisation epilogue shared by the tensor-core kernels (S7;
// the exact threshold map of reading Q23 written as one clamp + one multiply-add per column PAIR).
#pragma once
#include <stdint.h>

#include "unpack.cuh"

namespace dg {

__device__ __forceinline__ void store_codes32_ts(uint8_t *dp, uint32_t o0, uint32_t o1, int nbytes) {
#pragma unroll
    for (int b = 0; b < 8; ++b)
        if (b < nbytes) dp[b] = (uint8_t)((b < 4 ? o0 : o1) >> (8 * (b & 3)));
}

// 16-bit SIMD requant of 32 columns (S7; the exact threshold map of reading Q23 written as one
// clamp + one multiply-add per column PAIR).  r[i] = columns 2i | 2i+1 (tcgen05.ld pack::16b),
// na[i] = their offsets.  The code of lane j ends in bits [14,16) of that lane; PRMT gathers the
// four codes of 4 consecutive columns into the top bits of 4 bytes, a masked multiply by
// 2^18+2^12+2^6+1 moves them into the top byte in LSB-first order (the cross terms land below
// bit 24 without overlapping, or above bit 31), and two PRMT levels assemble 16 columns per word.
__device__ __forceinline__ uint2 requant16_32(const uint32_t (&r)[16], const uint32_t (&na)[16], uint32_t w2, uint32_t m, uint32_t c2) {
    uint32_t y[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) y[i] = __viaddmin_s16x2_relu(r[i], na[i], w2) * m + c2;
    uint32_t u[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) u[b] = (prmt_b32(y[2 * b], y[2 * b + 1], 0x7531u) & 0xC0C0C0C0u) * 0x41041u;
    const uint32_t lo = prmt_b32(prmt_b32(u[0], u[1], 0x0073u), prmt_b32(u[2], u[3], 0x0073u), 0x5410u);
    const uint32_t hi = prmt_b32(prmt_b32(u[4], u[5], 0x0073u), prmt_b32(u[6], u[7], 0x0073u), 0x5410u);
    return make_uint2(lo, hi);
}


}  // namespace dg
