/*
 * oracle.c — plain, slow, obviously-correct CPU reference for the DeepGEMM
 * (arXiv 2304.09049) 2-bit LUT GEMM / convolution hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_2304_09049_b200/) may include, link or call this file.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may use it.  It shares no header, helper, table or constant with the
 * CUDA path.
 *
 * Citation convention: "P:NNN" = line NNN of /root/reference/PAPER.md,
 * "S:NNN" = line NNN of /root/reference/SPEC.md, "BJ" = BASELINE.json,
 * "Qn" = the n-th reading in DESIGN.md §3 (ambiguity register).
 *
 * Every function is a direct transcription of the definition it cites:
 * plain nested loops in the paper's order, no blocking, no fusion, no
 * reordering.  Integer sums are carried in int64 and checked against the
 * int32 output range.
 */
#include <stdint.h>
#include <stddef.h>
#include <math.h>

/* ------------------------------------------------------------------------ */
/* Packed format (Fig. 1a caption, §3.1: several 2-bit values are
 * packed into one byte with shift/OR).  Layout reading (Q20,
 * S:129): code k of a row sits in byte k>>2, bits [2(k&3), 2(k&3)+1]
 * (LSB-first).  Rows are `ld` bytes apart.                                  */

/* Unpack `rows` x `K` codes from a packed buffer (oracle-side reader of the
 * documented format, used to check the GPU packer independently). */
void or_unpack_codes(const uint8_t *packed, int64_t rows, int64_t K, int64_t ld,
                     uint8_t *codes /* [rows][K] */)
{
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t k = 0; k < K; ++k) {
            uint8_t byte = packed[r * ld + (k / 4)];
            int shift = 2 * (int)(k % 4);
            codes[r * K + k] = (uint8_t)((byte >> shift) & 3);
        }
}

/* ------------------------------------------------------------------------ */
/* LUT-16 (§3.2): "The values stored in the LUT are all possible results
 * of w·a, with w ∈ {ω00,ω01,ω10,ω11} and a ∈ {α00,α01,α10,α11}".  The index is
 * the weight code concatenated above the activation code (Alg. 1 line 9,
 * P:235; reading Q7): T[(i<<2)|j] = wl[i] * al[j]. */
void or_build_lut16(const int32_t wl[4], const int32_t al[4], int32_t T[16])
{
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j)
            T[(i << 2) | j] = wl[i] * al[j];
}

/* ------------------------------------------------------------------------ */
/* LUT GEMM (Alg. 1; §3.1: unpack, concatenate into an index,
 * look the product up, sum).  BJ naming (reading Q1):
 *     C[m][n] = sum_{k<K} T[ (W[m][k] << 2) | A[k][n] ]
 * W codes are [M][K] row-major, A codes are [K][N] row-major, C is [M][N].
 * Returns 0, or -1 if any |C| does not fit int32 (reading Q8: exact int32
 * accumulation is normative). */
int or_lut_gemm(const uint8_t *W, const uint8_t *A, int64_t M, int64_t N, int64_t K,
                const int32_t T[16], int32_t *C)
{
    int overflow = 0;
    for (int64_t m = 0; m < M; ++m)
        for (int64_t n = 0; n < N; ++n) {
            int64_t acc = 0;
            for (int64_t k = 0; k < K; ++k) {
                int w = W[m * K + k] & 3;
                int a = A[k * N + n] & 3;
                int idx = (w << 2) | a;          /* Alg. 1 line 9 */
                acc += T[idx];                   /* Alg. 1 line 10 + reduction_sum */
            }
            if (acc > INT32_MAX || acc < INT32_MIN) overflow = 1;
            C[m * N + n] = (int32_t)acc;
        }
    return overflow ? -1 : 0;
}

/* ------------------------------------------------------------------------ */
/* b-bit LUT GEMM (P:183-184 §"Scalability to Larger Bitwidths", Table 2 at P:164-181: for b-bit
 * operands the index is the b-bit weight code concatenated above the b-bit activation code, a
 * 2b-bit index into a 2^(2b)-entry table: 64 entries for 3-bit, 256 for 4-bit):
 *     C[m][n] = sum_{k<K} T[ (W[m][k] << b) | A[k][n] ],   codes in [0, 2^b)
 * Same loop order and int64 / int32 check as or_lut_gemm (b = 2 is that function). */
int or_lut_gemm_bits(const uint8_t *W, const uint8_t *A, int64_t M, int64_t N, int64_t K, int32_t bits,
                     const int32_t *T /* [1 << (2*bits)] */, int32_t *C)
{
    int overflow = 0;
    const int mask = (1 << bits) - 1;
    for (int64_t m = 0; m < M; ++m)
        for (int64_t n = 0; n < N; ++n) {
            int64_t acc = 0;
            for (int64_t k = 0; k < K; ++k) {
                int w = W[m * K + k] & mask;
                int a = A[k * N + n] & mask;
                acc += T[(w << bits) | a];
            }
            if (acc > INT32_MAX || acc < INT32_MIN) overflow = 1;
            C[m * N + n] = (int32_t)acc;
        }
    return overflow ? -1 : 0;
}

/* ------------------------------------------------------------------------ */
/* Direct 2-D convolution over codes (the layer the paper lowers to an
 * (M,N,K) GEMM, §5.1), written as the textbook 7-loop definition, NOT
 * via im2col, so that it shares no logic with the GEMM lowering:
 *   out[b][ho][wo][co] = sum_{r<kh} sum_{s<kw} sum_{c<C}
 *        T[ (w[co][r][s][c] << 2) | x_code(b, ho*stride - pad + r, wo*stride - pad + s, c) ]
 * with x_code = pad_code outside the image (reading Q21).
 * x codes NHWC [B][H][Wd][C]; w codes [Cout][kh][kw][C]; out int32 NHWC
 * [B][Ho][Wo][Cout], Ho = (H + 2 pad - kh)/stride + 1 (same for Wo). */
int or_conv2d_direct(const uint8_t *x, const uint8_t *w, int32_t B, int32_t H, int32_t Wd,
                     int32_t C, int32_t Cout, int32_t kh, int32_t kw, int32_t stride,
                     int32_t pad, uint8_t pad_code, const int32_t T[16], int32_t *out)
{
    int overflow = 0;
    int32_t Ho = (H + 2 * pad - kh) / stride + 1;
    int32_t Wo = (Wd + 2 * pad - kw) / stride + 1;
    for (int32_t b = 0; b < B; ++b)
        for (int32_t ho = 0; ho < Ho; ++ho)
            for (int32_t wo = 0; wo < Wo; ++wo)
                for (int32_t co = 0; co < Cout; ++co) {
                    int64_t acc = 0;
                    for (int32_t r = 0; r < kh; ++r)
                        for (int32_t s = 0; s < kw; ++s)
                            for (int32_t c = 0; c < C; ++c) {
                                int32_t hi = ho * stride - pad + r;
                                int32_t wi = wo * stride - pad + s;
                                int a;
                                if (hi < 0 || hi >= H || wi < 0 || wi >= Wd)
                                    a = pad_code & 3;
                                else
                                    a = x[(((int64_t)b * H + hi) * Wd + wi) * C + c] & 3;
                                int wc = w[(((int64_t)co * kh + r) * kw + s) * C + c] & 3;
                                acc += T[(wc << 2) | a];
                            }
                    if (acc > INT32_MAX || acc < INT32_MIN) overflow = 1;
                    out[(((int64_t)b * Ho + ho) * Wo + wo) * Cout + co] = (int32_t)acc;
                }
    return overflow ? -1 : 0;
}

/* b-bit direct convolution (or_conv2d_direct with the b-bit index of P:183-184 / Table 2):
 *   out = sum_{r,s,c} T[(w << b) | x_code], out-of-image taps read pad_code. */
int or_conv2d_direct_bits(const uint8_t *x, const uint8_t *w, int32_t B, int32_t H, int32_t Wd,
                          int32_t C, int32_t Cout, int32_t kh, int32_t kw, int32_t stride,
                          int32_t pad, uint8_t pad_code, int32_t bits, const int32_t *T, int32_t *out)
{
    int overflow = 0;
    const int mask = (1 << bits) - 1;
    int32_t Ho = (H + 2 * pad - kh) / stride + 1;
    int32_t Wo = (Wd + 2 * pad - kw) / stride + 1;
    for (int32_t b = 0; b < B; ++b)
        for (int32_t ho = 0; ho < Ho; ++ho)
            for (int32_t wo = 0; wo < Wo; ++wo)
                for (int32_t co = 0; co < Cout; ++co) {
                    int64_t acc = 0;
                    for (int32_t r = 0; r < kh; ++r)
                        for (int32_t s = 0; s < kw; ++s)
                            for (int32_t c = 0; c < C; ++c) {
                                int32_t hi = ho * stride - pad + r;
                                int32_t wi = wo * stride - pad + s;
                                int a;
                                if (hi < 0 || hi >= H || wi < 0 || wi >= Wd)
                                    a = pad_code & mask;
                                else
                                    a = x[(((int64_t)b * H + hi) * Wd + wi) * C + c] & mask;
                                int wc = w[(((int64_t)co * kh + r) * kw + s) * C + c] & mask;
                                acc += T[(wc << bits) | a];
                            }
                    if (acc > INT32_MAX || acc < INT32_MIN) overflow = 1;
                    out[(((int64_t)b * Ho + ho) * Wo + wo) * Cout + co] = (int32_t)acc;
                }
    return overflow ? -1 : 0;
}

/* ------------------------------------------------------------------------ */
/* Integer requantisation (Eq. 1, with s·x realised as the exact
 * rational v·mult / 2^shift, reading Q11; round half away from zero,
 * reading Q5 / S:90; clip to [qmin,qmax], reading Q3/Q4):
 *     v    = acc + res + bias
 *     p    = v * mult                                  (exact, int64)
 *     q    = rhaz(p / 2^shift)
 *     code = clip(q + zp, qmin, qmax)
 * acc/res are [rows][cols] with leading dimension `ld` (res may be NULL);
 * bias may be NULL, else indexed bias[col] (bias_axis 0) or bias[row]
 * (bias_axis 1).  Codes out are one per byte, [rows][cols]. */
static int64_t or_rhaz(int64_t p, int32_t shift)
{
    /* p / 2^shift rounded half away from zero, written on the magnitude so
     * the tie rule is visibly symmetric */
    if (shift == 0) return p;
    int64_t half = (int64_t)1 << (shift - 1);
    if (p >= 0) return (p + half) >> shift;
    return -((-p + half) >> shift);
}

void or_requantize(const int32_t *acc, const int32_t *res, int64_t rows, int64_t cols, int64_t ld,
                   const int32_t *bias, int32_t bias_axis, int32_t mult, int32_t shift,
                   int32_t zp, int32_t qmin, int32_t qmax, uint8_t *codes)
{
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) {
            int64_t v = (int64_t)acc[r * ld + c];
            if (res) v += (int64_t)res[r * ld + c];
            if (bias) v += (int64_t)(bias_axis == 0 ? bias[c] : bias[r]);
            int64_t p = v * (int64_t)mult;
            int64_t q = or_rhaz(p, shift) + zp;
            if (q < qmin) q = qmin;
            if (q > qmax) q = qmax;
            codes[r * cols + c] = (uint8_t)q;
        }
}

/* ------------------------------------------------------------------------ */
/* Eq. 1 on floats: x_q = clip(round(s·x + z), qmin, qmax), round
 * half away from zero, s·x + z formed with one fused multiply-add
 * (reading Q22: removes the mul/add contraction ambiguity). */
void or_quantize(const float *x, int64_t n, float s, float z, int32_t qmin, int32_t qmax,
                 int32_t *q)
{
    for (int64_t i = 0; i < n; ++i) {
        float t = fmaf(s, x[i], z);
        float r = roundf(t);                 /* C roundf: half away from zero */
        int64_t v = (int64_t)r;
        if (v < qmin) v = qmin;
        if (v > qmax) v = qmax;
        q[i] = (int32_t)v;
    }
}

/* ------------------------------------------------------------------------ */
/* Freivalds check of a full C = LUTGEMM(W, A, T) output when the plain
 * triple loop is too slow.  For a random vector x:
 *   (C x)[m] = sum_n C[m][n] x[n]
 *            = sum_k sum_{a<4} T[(W[m][k]<<2)|a] * H[k][a],
 *   H[k][a]  = sum_n [A[k][n] == a] * x[n].
 * Exact in __int128.  A is given K-major as At[N][K] codes (the layout the
 * GPU operand uses) to avoid a transpose of a large array; C is [M][N] with
 * leading dimension ldc.  Returns the number of rows m where the two sides
 * differ (0 = consistent). */
int64_t or_freivalds_rows(const uint8_t *W, const uint8_t *At, const int32_t *C, int64_t ldc,
                          int64_t M, int64_t N, int64_t K, const int32_t T[16],
                          const int64_t *x, __int128 *H_scratch /* [K][4] */)
{
    for (int64_t k = 0; k < K; ++k)
        for (int a = 0; a < 4; ++a) H_scratch[k * 4 + a] = 0;
    for (int64_t n = 0; n < N; ++n)
        for (int64_t k = 0; k < K; ++k)
            H_scratch[k * 4 + (At[n * K + k] & 3)] += x[n];
    int64_t bad = 0;
    for (int64_t m = 0; m < M; ++m) {
        __int128 lhs = 0, rhs = 0;
        for (int64_t n = 0; n < N; ++n) lhs += (__int128)C[m * ldc + n] * x[n];
        for (int64_t k = 0; k < K; ++k) {
            int w = W[m * K + k] & 3;
            for (int a = 0; a < 4; ++a) rhs += (__int128)T[(w << 2) | a] * H_scratch[k * 4 + a];
        }
        if (lhs != rhs) ++bad;
    }
    return bad;
}

/* ------------------------------------------------------------------------ */
/* Freivalds check of a whole convolution output (the conv of
 * or_conv2d_direct) when the direct loops are too slow for a full
 * batch.  For a random weight r[p] per output pixel p = (b, ho, wo):
 *   sum_p r[p] out[p][co]
 *     = sum_p r[p] sum_{i,j,c} T[(w[co][i][j][c] << 2) | x_code(p, i, j, c)]
 *     = sum_{i,j,c} sum_{a<4} T[(w[co][i][j][c] << 2) | a] * H[i][j][c][a],
 *   H[i][j][c][a] = sum_p r[p] [x_code(p, i, j, c) == a]
 * (x_code = pad_code outside the image, as in or_conv2d_direct).  Exact in
 * __int128.  out is int32 NHWC [B][Ho][Wo][Cout] with row pitch ldo elements;
 * r has B*Ho*Wo entries; H_scratch holds kh*kw*C*4 __int128.  Returns the
 * number of output channels co where the two sides differ (0 = consistent). */
int64_t or_conv_freivalds(const uint8_t *x, const uint8_t *w, int32_t B, int32_t H, int32_t Wd,
                          int32_t C, int32_t Cout, int32_t kh, int32_t kw, int32_t stride,
                          int32_t pad, uint8_t pad_code, const int32_t T[16], const int32_t *out,
                          int64_t ldo, const int64_t *r, __int128 *H_scratch)
{
    int32_t Ho = (H + 2 * pad - kh) / stride + 1;
    int32_t Wo = (Wd + 2 * pad - kw) / stride + 1;
    int64_t ntap = (int64_t)kh * kw * C;
    for (int64_t t = 0; t < ntap * 4; ++t) H_scratch[t] = 0;
    for (int32_t b = 0; b < B; ++b)
        for (int32_t ho = 0; ho < Ho; ++ho)
            for (int32_t wo = 0; wo < Wo; ++wo) {
                int64_t p = ((int64_t)b * Ho + ho) * Wo + wo;
                for (int32_t i = 0; i < kh; ++i)
                    for (int32_t j = 0; j < kw; ++j)
                        for (int32_t c = 0; c < C; ++c) {
                            int32_t hi = ho * stride - pad + i;
                            int32_t wi = wo * stride - pad + j;
                            int a;
                            if (hi < 0 || hi >= H || wi < 0 || wi >= Wd)
                                a = pad_code & 3;
                            else
                                a = x[(((int64_t)b * H + hi) * Wd + wi) * C + c] & 3;
                            H_scratch[(((int64_t)i * kw + j) * C + c) * 4 + a] += r[p];
                        }
            }
    int64_t bad = 0;
    int64_t P = (int64_t)B * Ho * Wo;
    for (int32_t co = 0; co < Cout; ++co) {
        __int128 lhs = 0, rhs = 0;
        for (int64_t p = 0; p < P; ++p) lhs += (__int128)out[p * ldo + co] * r[p];
        for (int32_t i = 0; i < kh; ++i)
            for (int32_t j = 0; j < kw; ++j)
                for (int32_t c = 0; c < C; ++c) {
                    int wc = w[(((int64_t)co * kh + i) * kw + j) * C + c] & 3;
                    for (int a = 0; a < 4; ++a)
                        rhs += (__int128)T[(wc << 2) | a] * H_scratch[(((int64_t)i * kw + j) * C + c) * 4 + a];
                }
        if (lhs != rhs) ++bad;
    }
    return bad;
}

/* ------------------------------------------------------------------------ */
/* LUT GEMM over a FLOAT-valued table (§5.3: "The LUT can store either integer or
 * floating-point values", e.g. the products of a non-uniform quantiser's levels):
 *     C[m][n] = sum_{k<K} T[(W[m][k] << 2) | A[k][n]]        (T double, summed in double)
 * Same loops and index as or_lut_gemm (Alg. 1); the sum is carried in fp64 in k
 * order, so it is the exact value up to K * 2^-53 * sum|T| (reading Q24). */
void or_lut_gemm_f64(const uint8_t *W, const uint8_t *A, int64_t M, int64_t N, int64_t K,
                     const double T[16], double *C)
{
    for (int64_t m = 0; m < M; ++m)
        for (int64_t n = 0; n < N; ++n) {
            double acc = 0.0;
            for (int64_t k = 0; k < K; ++k) {
                int w = W[m * K + k] & 3;
                int a = A[k * N + n] & 3;
                acc += T[(w << 2) | a];
            }
            C[m * N + n] = acc;
        }
}
