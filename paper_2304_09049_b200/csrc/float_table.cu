// float_table.cu — LUT GEMM over a FLOAT-valued 16-entry table (§5.3: "The LUT can store
// either integer or floating-point values", e.g. the products of a non-uniform quantiser's levels,
// P:102-103), on the int8 tensor cores:
//
//   C[m][n] = sum_{k<K} T[(W[m][k] << 2) | A[k][n]]                                  (Alg. 1)
//
// The table is written in 24-bit fixed point, Ti = rne(T * 2^s) with 2^s the largest power of two
// that keeps max|Ti| <= 127 * (2^16 + 2^8 + 1), and split into three balanced int8 digits,
// Ti = d2 * 2^16 + d1 * 2^8 + d0.  Each digit table is an arbitrary int8 table, so its LUT sum is
// an exact int8 dot product in the one-hot form (dg_lut_gemm_onehot: K' = 4K); the three digit
// GEMMs run as ONE tensor-core GEMM with the three table-column operands stacked along N, and the
// combine kernel forms (acc2 * 2^16 + acc1 * 2^8 + acc0) * 2^-s exactly in fp64 (an integer below
// 2^53) before the single rounding to fp32.  Error bound (reading Q24):
//   |C - sum_k T| <= K * max|T| / Q + 2^-24 |sum_k T|,   Q = 127 * (2^16 + 2^8 + 1).
#include <math.h>
#include <string.h>

#include "common.cuh"

namespace dg {
namespace {

constexpr int64_t F32_Q = 127 * (65536 + 256 + 1);   // largest |Ti| with three balanced int8 digits

__global__ void combine_digits_kernel(const int32_t *__restrict__ acc, int64_t M, int64_t N, double scale,
                                      float *__restrict__ C, int64_t ldc) {
    const int64_t total = M * N;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = i / N, n = i - m * N;
        const int32_t *row = acc + m * 3 * N;
        const double v = ((double)row[2 * N + n] * 65536.0 + (double)row[N + n] * 256.0 + (double)row[n]) * scale;
        C[m * ldc + n] = (float)v;
    }
}

}  // namespace

// host: fixed-point scale and the three digit tables of a float table; false if every entry is 0
bool float_table_digits(const float T[16], int32_t digits[3][16], int32_t *s_out) {
    double tmax = 0;
    for (int e = 0; e < 16; ++e) tmax = fabs((double)T[e]) > tmax ? fabs((double)T[e]) : tmax;
    int s = 0;
    if (tmax > 0) {
        int ex = 0;
        frexp(tmax, &ex);   // tmax in [2^(ex-1), 2^ex)
        s = 23 - ex;        // tmax * 2^s < 2^23 ...
        while (tmax * ldexp(1.0, s) > (double)F32_Q) --s;      // ... and <= Q
        while (tmax * ldexp(1.0, s + 1) <= (double)F32_Q) ++s;
    }
    for (int e = 0; e < 16; ++e) {
        int64_t ti = (int64_t)nearbyint(ldexp((double)T[e], s));   // round half to even
        int64_t d0 = ((ti % 256) + 256 + 128) % 256 - 128;
        int64_t t1 = (ti - d0) / 256;
        int64_t d1 = ((t1 % 256) + 256 + 128) % 256 - 128;
        int64_t d2 = (t1 - d1) / 256;
        digits[0][e] = (int32_t)d0;
        digits[1][e] = (int32_t)d1;
        digits[2][e] = (int32_t)d2;
    }
    *s_out = s;
    return tmax > 0;
}

int64_t lut_gemm_f32_workspace(int64_t M, int64_t N, int64_t K) {
    return (M * onehot_ld(K) + 127) / 128 * 128 + 3 * N * tcols_ld(K) + (M * 3 * N * 4 + 127) / 128 * 128 + 384;
}

dg_status lut_gemm_f32(const uint8_t *W, int64_t ldw, const uint8_t *At, int64_t lda, int64_t M, int64_t N, int64_t K,
                       const float T[16], float *C, int64_t ldc, void *ws, size_t ws_bytes, cudaStream_t st) {
    int32_t dig[3][16];
    int32_t s = 0;
    const bool nonzero = float_table_digits(T, dig, &s);
    const int64_t l1 = onehot_ld(K), lt = tcols_ld(K);
    uint8_t *w1h = (uint8_t *)(((uintptr_t)ws + 127) & ~(uintptr_t)127);
    int8_t *atc = (int8_t *)(((uintptr_t)(w1h + M * l1) + 127) & ~(uintptr_t)127);
    int32_t *acc = (int32_t *)(((uintptr_t)(atc + 3 * N * lt) + 127) & ~(uintptr_t)127);
    if ((uint8_t *)(acc + M * 3 * N) > (uint8_t *)ws + ws_bytes) return DG_ERR_WORKSPACE;
    dg_status r = expand_onehot(W, M, K, ldw, w1h, l1, st);
    for (int d = 0; d < 3 && r == DG_OK; ++d) r = expand_tcols(At, N, K, lda, dig[d], atc + d * N * lt, lt, st);
    if (r != DG_OK) return r;
    // the three digit GEMMs as one: rows of the stacked table-column operand [3N][lt]
    const int32_t pl[4] = {0, 1, 0, 0}, ql[4] = {128, 0, 0, 0};   // (ql only bounds |acc| <= 4K * 128)
    r = lut_gemm_ts(w1h, l1, atc, lt, M, 3 * N, 4 * K, pl, ql, acc, 3 * N, nullptr, st);
    if (r != DG_OK) return r;
    int64_t blocks = (M * N + 255) / 256;
    if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
    combine_digits_kernel<<<(int)blocks, 256, 0, st>>>(acc, M, N, nonzero ? ldexp(1.0, -s) : 0.0, C, ldc);
    set_last_kernel("f32 table: one-hot 3-digit ts + combine");
    return launch_status();
}

}  // namespace dg
