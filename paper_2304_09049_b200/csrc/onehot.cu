// onehot.cu — LUT-16 GEMM for NON-product tables on the int8 tensor cores (SURVEY §8(f) rank 3,
// the "one-hot K' = 4K formulation").
//
// Any 16-entry table splits over the weight code (Alg. 1's lookup):
//     T[(w << 2) | a] = sum_{i=0..3} [w == i] * T[(i << 2) | a]
// so  C[m][n] = sum_k T[(W[m][k] << 2) | A[k][n]] = sum_{k' < 4K} P'[m][k'] * Q'[n][k']  with
//     P'[m][4k + i] = [W[m][k] == i]         (0/1: a 2-bit code, identity level)
//     Q'[n][4k + i] = T[(i << 2) | A[k][n]]   (an int8 entry)
// an int8 dot product of length 4K, exact in s32.  Both operands are produced once from packed
// codes by the two kernels below; the GEMM itself is the TS kernel (lut_gemm_ts.cu) with K' = 4K.
// For product tables the plain tc path (K, levels) does a quarter of this work.
#include "common.cuh"
#include "unpack.cuh"

namespace dg {
namespace {

// P': packed weights [rows][ld] -> packed one-hot codes [rows][ld_out]: original code k becomes
// byte k = 1 << (2 * code) (the codes of k' = 4k..4k+3 are [code == 0], .., [code == 3]); bytes
// for k >= K are 0.  One thread per 4 input bytes (16 codes -> 16 output bytes).
__global__ void expand_onehot_kernel(const uint8_t *__restrict__ w, int64_t rows, int64_t K, int64_t ld,
                                     uint8_t *__restrict__ out, int64_t ld_out) {
    const int64_t groups = ld_out / 16;
    const int64_t total = rows * groups;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / groups, g = i - r * groups;
        const uint32_t x = 4 * g + 4 <= ld ? *reinterpret_cast<const uint32_t *>(w + r * ld + 4 * g) : 0u;
        uint32_t o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t v = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int j = 4 * q + b;                 // code j of the 16
                const uint32_t c = (x >> (2 * j)) & 3u;
                if (16 * g + j < K) v |= (1u << (2 * c)) << (8 * b);
            }
            o[q] = v;
        }
        *reinterpret_cast<uint4 *>(out + r * ld_out + 16 * g) = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

// Q': packed activations [rows][ld] -> int8 [rows][ld_out] of T[(i << 2) | a] at k' = 4k + i, in
// the TS kernel's unpack order (the 16 k' of a 32-bit word as 0,2,..,14,1,3,..,15, unpack.cuh),
// 0 for k >= K.  One thread per 16 output bytes (4 original codes).
__global__ void expand_tcols_kernel(const uint8_t *__restrict__ a, int64_t rows, int64_t K, int64_t ld,
                                    uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3, int8_t *__restrict__ out,
                                    int64_t ld_out) {
    const uint32_t tab[4] = {t0, t1, t2, t3};   // tab[a] byte i = T[(i << 2) | a]
    const int64_t groups = ld_out / 16;
    const int64_t total = rows * groups;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / groups, g = i - r * groups;   // output bytes = k' in [16g, 16g + 16)
        const uint32_t x = g < ld ? a[r * ld + g] : 0u;     // original codes k = 4g .. 4g + 3
        uint32_t o[4] = {0, 0, 0, 0};
#pragma unroll
        for (int b = 0; b < 16; ++b) {
            const int kp = b < 8 ? 2 * b : 2 * (b - 8) + 1;   // k' offset stored at byte b
            const int kk = kp >> 2, ii = kp & 3;
            const uint32_t c = (x >> (2 * kk)) & 3u;
            const uint32_t v = (4 * g + kk < K) ? ((tab[c] >> (8 * ii)) & 0xFFu) : 0u;
            o[b >> 2] |= v << (8 * (b & 3));
        }
        *reinterpret_cast<uint4 *>(out + r * ld_out + 16 * g) = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

// 4-bit operands through the 2-bit tensor-core path (Table 2):
// a 4-bit activation code a with identity level is the two 2-bit digits a = a_l + 4 a_h, and a
// packed 4-bit row (code k in nibble k&1 of byte k>>1, low first) IS a packed 2-bit row of the
// digits at k' = 2k (a_l) and 2k + 1 (a_h).  So sum_k wl[w_k] a_k = sum_{k'} digit[k'] Q'[k'] with
// Q'[2k] = wl[w_k], Q'[2k + 1] = 4 wl[w_k]: the weights' side, built here as int8 in the
// tensor-core operand order (unpack.cuh), 0 for k >= K.  One thread per 16 output bytes.
struct Lev16 {
    int8_t v[16];
};
__global__ void expand_digits4_kernel(const uint8_t *__restrict__ w4, int64_t rows, int64_t K, int64_t ld,
                                      const __grid_constant__ Lev16 sl4, int8_t *__restrict__ out, int64_t ld_out) {
    const int8_t *sl = sl4.v;
    const int64_t groups = ld_out / 16;
    const int64_t total = rows * groups;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / groups, g = i - r * groups;   // k' in [16g, 16g + 16): codes k = 8g .. 8g + 7
        uint32_t o[4] = {0, 0, 0, 0};
#pragma unroll
        for (int b = 0; b < 16; ++b) {
            const int kp = b < 8 ? 2 * b : 2 * (b - 8) + 1;
            const int64_t k = 8 * g + (kp >> 1);
            int32_t v = 0;
            if (k < K) {
                const uint32_t code = (w4[r * ld + (k >> 1)] >> (4 * (k & 1))) & 15u;
                v = (kp & 1) ? 4 * sl[code] : sl[code];
            }
            o[b >> 2] |= ((uint32_t)v & 0xFFu) << (8 * (b & 3));
        }
        *reinterpret_cast<uint4 *>(out + r * ld_out + 16 * g) = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

// 4-bit codes, any 256-entry table (Table 2: the 2b-bit index into a 2^(2b)-entry
// LUT; 3-bit tables are 4-bit tables over codes 0..7): the one-hot split over the 16 weight codes,
//     P'[m][16k + i] = [W[m][k] == i],   Q'[n][16k + i] = T[(i << 4) | A[k][n]],   K' = 16K.
// P': packed 4-bit weights [rows][ld] -> packed 2-bit one-hot codes, 4 bytes per original code
// (the 32-bit word 1 << (2 code)); one thread per 4 original codes (16 output bytes).
__global__ void expand_onehot4_kernel(const uint8_t *__restrict__ w4, int64_t rows, int64_t K, int64_t ld,
                                      uint8_t *__restrict__ out, int64_t ld_out) {
    const int64_t groups = ld_out / 16;
    const int64_t total = rows * groups;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / groups, g = i - r * groups;   // original codes k = 4g .. 4g + 3
        uint32_t o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t k = 4 * g + q;
            const uint32_t c = k < K ? (w4[r * ld + (k >> 1)] >> (4 * (k & 1))) & 15u : 0u;
            o[q] = k < K ? 1u << (2 * c) : 0u;
        }
        *reinterpret_cast<uint4 *>(out + r * ld_out + 16 * g) = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

// Q': packed 4-bit activations [rows][ld] -> int8 [rows][ld_out] of T[(i << 4) | a] at k' = 16k + i,
// in the TS kernel's unpack order (the 16 k' of original code k as 0,2,..,14,1,3,..,15), 0 for
// k >= K.  One thread per original code (16 output bytes).
struct Tab256 {
    int8_t v[256];
};
__global__ void expand_tcols4_kernel(const uint8_t *__restrict__ a4, int64_t rows, int64_t K, int64_t ld,
                                     const __grid_constant__ Tab256 tab, int8_t *__restrict__ out, int64_t ld_out) {
    const int64_t groups = ld_out / 16;
    const int64_t total = rows * groups;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / groups, k = i - r * groups;
        const uint32_t x = k < K ? (a4[r * ld + (k >> 1)] >> (4 * (k & 1))) & 15u : 0u;
        uint32_t o[4] = {0, 0, 0, 0};
#pragma unroll
        for (int b = 0; b < 16; ++b) {
            const int ii = b < 8 ? 2 * b : 2 * (b - 8) + 1;   // weight code i stored at byte b
            const uint32_t v = k < K ? (uint32_t)(uint8_t)tab.v[(ii << 4) | x] : 0u;
            o[b >> 2] |= v << (8 * (b & 3));
        }
        *reinterpret_cast<uint4 *>(out + r * ld_out + 16 * k) = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

int64_t grid_for(int64_t work) {
    int64_t blocks = (work + 255) / 256;
    const int64_t cap = (int64_t)num_sms() * 8;
    return blocks > cap ? cap : (blocks < 1 ? 1 : blocks);
}

}  // namespace

dg_status expand_digits4(const uint8_t *w4, int64_t rows, int64_t K, int64_t ld, const int32_t levels[16], int8_t *out,
                         int64_t ld_out, cudaStream_t st) {
    Lev16 l;   // the 16 levels travel by value in the kernel parameters
    for (int i = 0; i < 16; ++i) l.v[i] = (int8_t)levels[i];
    if (rows == 0) return DG_OK;
    expand_digits4_kernel<<<(int)grid_for(rows * (ld_out / 16)), 256, 0, st>>>(w4, rows, K, ld, l, out, ld_out);
    return launch_status();
}

int64_t onehot_ld(int64_t K) { return (K + 15) / 16 * 16; }
int64_t onehot4_ld(int64_t K) { return (4 * K + 15) / 16 * 16; }
int64_t tcols4_ld(int64_t K) { return expand_ld(16 * K); }

dg_status expand_onehot4(const uint8_t *w4, int64_t rows, int64_t K, int64_t ld, uint8_t *out, int64_t ld_out,
                         cudaStream_t st) {
    if (rows == 0) return DG_OK;
    expand_onehot4_kernel<<<(int)grid_for(rows * (ld_out / 16)), 256, 0, st>>>(w4, rows, K, ld, out, ld_out);
    return launch_status();
}

dg_status expand_tcols4(const uint8_t *a4, int64_t rows, int64_t K, int64_t ld, const int32_t table[256], int8_t *out,
                        int64_t ld_out, cudaStream_t st) {
    Tab256 t;   // the table travels by value in the kernel parameters
    for (int e = 0; e < 256; ++e) t.v[e] = (int8_t)table[e];
    if (rows == 0) return DG_OK;
    expand_tcols4_kernel<<<(int)grid_for(rows * (ld_out / 16)), 256, 0, st>>>(a4, rows, K, ld, t, out, ld_out);
    return launch_status();
}
int64_t tcols_ld(int64_t K) { return expand_ld(4 * K); }

dg_status expand_onehot(const uint8_t *w, int64_t rows, int64_t K, int64_t ld, uint8_t *out, int64_t ld_out,
                        cudaStream_t st) {
    if (rows == 0) return DG_OK;
    expand_onehot_kernel<<<(int)grid_for(rows * (ld_out / 16)), 256, 0, st>>>(w, rows, K, ld, out, ld_out);
    return launch_status();
}

dg_status expand_tcols(const uint8_t *a, int64_t rows, int64_t K, int64_t ld, const int32_t entries[16], int8_t *out,
                       int64_t ld_out, cudaStream_t st) {
    uint32_t tab[4] = {0, 0, 0, 0};
    for (int c = 0; c < 4; ++c)
        for (int i = 0; i < 4; ++i) tab[c] |= ((uint32_t)entries[(i << 2) | c] & 0xFFu) << (8 * i);
    if (rows == 0) return DG_OK;
    expand_tcols_kernel<<<(int)grid_for(rows * (ld_out / 16)), 256, 0, st>>>(a, rows, K, ld, tab[0], tab[1], tab[2],
                                                                             tab[3], out, ld_out);
    return launch_status();
}

}  // namespace dg
