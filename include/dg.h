/*
 * dg.h — C ABI of the B200-native 2-bit LUT GEMM / convolution library
 * (libdg.so), after DeepGEMM, arXiv 2304.09049.
 *
 * Citation convention: "P:NNN" = line NNN of the paper text,
 * "S:NNN" = line NNN of SPEC.md, "BJ" = BASELINE.json, "Qn" = reading n of
 * DESIGN.md §3.
 *
 * ---------------------------------------------------------------------------
 * Conventions (all calls)
 *  - Every call returns dg_status.  No C++ exception crosses the ABI.
 *  - Pointers prefixed d_ are DEVICE pointers owned by the caller; the library
 *    never allocates, frees or synchronises.  Workspace needs are queried
 *    with *_workspace_size.  Device calls are asynchronous on `stream` (a
 *    cudaStream_t passed as void*, NULL = legacy default stream).
 *  - Validation reads no device memory: out-of-range codes inside device
 *    buffers are masked with &3 (and counted in d_err_count where offered).
 *  - Codes are unsigned 2-bit patterns 0..3.  Signed levels exist only in
 *    the level/product tables (reading Q2).
 *
 * Packed format (Fig. 1a caption, §3.1: 2-bit values packed into
 * bytes with shift/OR; bit layout reading Q20 = S:129):
 *  - row-major; each row holds K codes in ceil(K/4) bytes; code k of a row
 *    sits in byte k>>2, bits [2(k&3), 2(k&3)+1] (LSB first);
 *  - rows are `ld` bytes apart, ld >= ceil(K/4), ld % 16 == 0 (so every row
 *    starts 16-byte aligned for 128-bit loads and TMA);
 *  - codes k in [K, 4*ld) MUST be 0.  dg_pack_* and dg_im2col write them as
 *    0; the GEMM kernels rely on it and correct for them exactly (Q10).
 *
 * GEMM orientation (BJ naming, reading Q1): C[m][n] = sum_{k<K} T[(W[m][k]<<2) | A[k][n]]
 *  with both operands stored K-major: W as [M][ldw] packed rows, A as its
 *  transpose At [N][lda] packed rows (an im2col row = one output pixel).
 * ---------------------------------------------------------------------------
 */
#ifndef DG_H_
#define DG_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define DG_API __attribute__((visibility("default")))
#else
#define DG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t dg_status;
#define DG_OK 0
#define DG_ERR_INVALID_ARG (-1)  /* null pointer, bad enum, misaligned ld          */
#define DG_ERR_SHAPE (-2)        /* non-positive / inconsistent dimensions          */
#define DG_ERR_RANGE (-3)        /* parameter outside its documented range          */
#define DG_ERR_OVERFLOW (-4)     /* table entry does not fit entry_bits, or the
                                    worst-case |accumulator| reaches 2^31           */
#define DG_ERR_UNSUPPORTED (-5)  /* e.g. tc variant forced on a non-product table   */
#define DG_ERR_CUDA (-6)         /* a CUDA launch / driver call failed              */
#define DG_ERR_WORKSPACE (-7)    /* workspace too small                             */

/* Static string for a status code (never NULL). */
DG_API const char *dg_status_string(dg_status s);

/* ABI version of this header (bumped on any signature change). */
#define DG_ABI_VERSION 4
DG_API int32_t dg_abi_version(void);

/* Number of CUDA kernels this library has enqueued since it was loaded (all
 * entry points, all streams; a launch recorded into a CUDA graph under stream
 * capture counts once, at capture).  Process-wide, thread-safe; for the
 * benchmark's launch count (kernels per step = difference across one step). */
DG_API uint64_t dg_kernel_launches(void);

/* ---------------------------------------------------------------------------
 * Runtime options (process-wide; every call reads them when it dispatches, so a change
 * applies to the next call).  They select among kernel instances that compute the SAME
 * result (ablations, tests that force an instance); none changes any output bit.
 * Defaults are the tuned dispatch; the DG_* environment variables of DESIGN.md §6.1 set
 * the initial values.  DG_ERR_INVALID_ARG for an unknown name.
 *   "win"       0 auto, 1 force the shifted-window kernel for every 3x3/s1/p1 conv with
 *               C in {64,128,256}, -1 never                                    (default 0)
 *   "win128"    C = 128 tile mode of the window kernel in auto dispatch       (1)
 *   "wpair"     window pair mode (one window feeds two row blocks)           (1)
 *   "asm"       short-K wide tiles with the A operand in shared memory       (1)
 *   "bn256"     128x256 tiles for long K                                     (1)
 *   "bn256_k"   minimum K (codes) for the 128x256 tiles                      (512)
 *   "kst"       codes per pipeline stage: 0 auto, 128 force 128-code stages  (0)
 *   "bn64_short" short-K layers with Cout > 64 on 64-wide tiles              (0)
 *   "splitk"    split-K for few-tile long-K GEMMs when workspace is given    (1)
 *   "f16"       16-bit SIMD requant epilogue (else the 32-bit threshold path)(1)
 *   "bres"      weight tiles resident in shared memory when they fit         (1)
 *   "pdl"       programmatic dependent launch of the GEMM kernels            (1)
 *   "early_weights"  the *_prepared calls may read their expanded weights and bias
 *               BEFORE waiting for the previous kernel on the stream (programmatic
 *               dependent launch: their prologue then overlaps that kernel's tail).
 *               Only correct when neither was written by a kernel still in flight
 *               on the stream (e.g. weights prepared at setup and synchronised).   (0)
 *   "f4conv"    route qualifying product-table layers to the block-scaled FP4 kernel (1)
 *   "em"        epilogue arrangement of the short-K wide kernel: 0 groups own alternate tiles,
 *               1 groups split each tile's columns, 2 epilogue warps first in scheduling
 *               priority, 3 both                                            (0)
 *   "tma_store" int32 output tiles through the TMA tensor store (staging in shared memory)
 *               instead of per-lane row stores, where the instance has room (1)
 *   "unp"       unpack warps of the 128x256 long-K int8 instance: 8, 12 or 16 (8)
 *   "f4_unp"    unpack warps of the FP4 conv kernel: 0 auto, 4 or 8         (0)
 *   "f4_epi"    epilogue warps of the FP4 conv kernel: 0 auto, 4 or 8       (0)
 *   "f4_bn"     FP4 conv tile width: 0 auto (256 when it divides Cout), 128, 256 (0)
 *   "f4_omma"   FP4 conv accumulators start from an origin MMA (one per tile) instead of
 *               tensor-memory reset stores                                   (1)
 *   "offs"      short-K shared-memory-A tiles start their accumulators at the columns' 16-bit
 *               requant offsets through one extra MMA (no offset loads in the epilogue)  (1)
 *   "bmc"       streamed-B GEMM/conv tiles: B stages multicast across 2-CTA clusters when the
 *               tile walk pairs row-adjacent tiles of one column block       (0)
 *   "skfuse"    split-K: the GEMM kernel sums its slices itself after a grid-wide barrier
 *               (cooperative launch) instead of a second reduce kernel       (0)
 *   "f4_ct"     FP4 conv: 2 = two CTAs per SM for the 128-wide tiles        (0)
 *   "f4_win"    FP4 conv: shifted-window mode for direct 3x3 / stride 1 / pad 1 convs over
 *               64 or 128 channels: 2 where the weights stay resident (one column block whose
 *               stages fit the B ring), 1 always, 0 never                    (2)
 *   "f4_wbres"  FP4 conv shifted window: all weight stages resident in shared memory (loaded
 *               once per CTA, one MMA hand-off per tile) when the layer is one column block (1)
 *   "f4_i2c"    FP4 conv: strided 1x1 convs (downsample) read their pixels through an
 *               im2col-mode TMA tensor map (element strides = the conv stride) on the direct
 *               path instead of the per-thread gather                        (1)
 *   "f4_w1x1"   FP4 conv: 1x1 stride-1 convs into 64 / 128 channels as window pairs (a
 *               pair's 256 pixel rows are the shared-memory A window): 1 over 64 input
 *               channels, 2 over 64 / 128 / 256, 0 never                    (1)
 *   "f4_wpair"  FP4 conv shifted window with resident 64 / 128-wide tiles: one window of 256 padded
 *               pixels + halo feeds two 128-row blocks into two accumulators (1)
 */
DG_API dg_status dg_set_option(const char *name, int64_t value);
DG_API dg_status dg_get_option(const char *name, int64_t *value);
DG_API dg_status dg_reset_options(void);   /* back to the defaults (environment ignored) */

/* Tag of the GEMM/conv kernel instance the CALLING THREAD launched last (static storage,
 * never NULL, "" before the first launch), e.g. "ts bn=128 epi=4 unp=8 kst=128 win nwin=2
 * wpair=0 ...": lets tests assert which instance computed a result. */
DG_API const char *dg_last_kernel(void);

/* ---------------------------------------------------------------------------
 * S4 — LUT build.  LUT-16 (§3.2): "The values stored in the LUT are all
 * possible results of w·a"; index = weight code concatenated above the
 * activation code (Alg. 1 line 9; reading Q7):
 *        entries[(i<<2)|j] = wl[i] * al[j].
 * Passed BY VALUE (by pointer to a host struct) to the GEMM calls.
 */
typedef struct {
    int32_t entries[16];  /* T[(w<<2)|a], sign-extended                               */
    int32_t entry_bits;   /* 8 | 16 | 32: declared storage width of the entries       */
    int32_t is_product;   /* 1 iff entries == wl (x) al exactly (enables the tc path)  */
    int32_t wl[4];        /* weight levels per code   (valid iff is_product)          */
    int32_t al[4];        /* activation levels per code (valid iff is_product)        */
} dg_lut;

/* Host.  Builds the product table from integer levels.  entry_bits must be 8,
 * 16 or 32; DG_ERR_OVERFLOW if any product does not fit a signed integer of
 * that width ("will not overflow 8 bits", is enforced). */
DG_API dg_status dg_build_lut(const int32_t wl[4], const int32_t al[4], int32_t entry_bits, dg_lut *out);

/* Host.  Wraps an arbitrary 16-entry table (LUT-16 with any precomputed
 * entries, §5.3 "flexibility"); is_product is detected exactly
 * (entries == wl (x) al for some integer levels is NOT searched: is_product=0). */
DG_API dg_status dg_lut_from_table(const int32_t entries[16], int32_t entry_bits, dg_lut *out);

/* Bytes per packed row for K codes: roundup(ceil(K/4), 16). */
DG_API int64_t dg_packed_ld(int64_t K);

/* ---------------------------------------------------------------------------
 * S1/S2 — packing (Fig. 1a).  d_codes is [rows][ld_codes] bytes,
 * one code per byte (values > 3 are masked with &3 and counted into
 * *d_err_count when it is non-NULL); d_packed is [rows][ld] in the packed
 * format above, zero-filled beyond K.  dg_pack_weights is the same operation
 * for the (offline) weight operand.                                   */
DG_API dg_status dg_pack_codes(const uint8_t *d_codes, int64_t rows, int64_t K, int64_t ld_codes,
                        uint8_t *d_packed, int64_t ld, int32_t *d_err_count, void *stream);
DG_API dg_status dg_pack_weights(const uint8_t *d_codes, int64_t rows, int64_t K, int64_t ld_codes,
                          uint8_t *d_packed, int64_t ld, int32_t *d_err_count, void *stream);

/* Device unpack (inverse of pack; test/debug aid): d_codes [rows][K]. */
DG_API dg_status dg_unpack_codes(const uint8_t *d_packed, int64_t rows, int64_t K, int64_t ld,
                          uint8_t *d_codes, void *stream);

/* S2 — Eq. 1 activation quantisation + pack:
 *      q    = clip(round(fma(scale, x, zero_point)), qmin, qmax)
 *      code = q - qmin                (offset-binary code, reading Q2)
 * round = half away from zero (Q5); requires 0 <= qmax - qmin <= 3.
 * d_x is fp32 [rows][K] (row stride K); output packed [rows][ld].           */
DG_API dg_status dg_quantize_pack_activations(const float *d_x, int64_t rows, int64_t K, float scale,
                                       float zero_point, int32_t qmin, int32_t qmax,
                                       uint8_t *d_packed, int64_t ld, void *stream);

/* ---------------------------------------------------------------------------
 * S3 — im2col over packed NHWC codes (the conv -> (M,N,K) GEMM lowering the
 * paper benchmarks on, §5.1).  d_x is [B][H][W][C/4] packed bytes
 * (C % 4 == 0: channels padded by the caller); row r = (b*Ho + ho)*Wo + wo of
 * d_cols ([B*Ho*Wo][ld]) holds the codes x(b, ho*stride-pad+r', wo*stride-pad+s', c)
 * in (r', s', c) order with c fastest, K = kh*kw*C; out-of-image taps hold
 * pad_code (reading Q21).                                                   */
DG_API dg_status dg_im2col(const uint8_t *d_x, int32_t B, int32_t H, int32_t W, int32_t C, int32_t kh,
                    int32_t kw, int32_t stride, int32_t pad, uint8_t pad_code, uint8_t *d_cols,
                    int64_t ld, void *stream);

/* ---------------------------------------------------------------------------
 * S7 — integer requantisation (Eq. 1 applied to the int32 accumulator with
 * s realised as mult*2^-shift, reading Q11; Q5 tie rule):
 *      v    = acc + res + bias
 *      q    = clip(rhaz(v*mult / 2^shift) + zp, qmin, qmax)      (int64 exact)
 *      code = q - qmin                                           (0 <= qmax-qmin <= 3)
 * where res = res_int32[r][c]  (d_res, a downsample shortcut's accumulator)
 *          or res_levels[res_code[r][c]] * res_mult (d_res_codes, identity
 *             shortcut over packed codes, reading Q13), and bias = bias[c]
 * (bias_axis 0) or bias[r] (bias_axis 1).  0 <= shift <= 62.                 */
typedef struct {
    int32_t mult, shift, zp, qmin, qmax;
    const int32_t *d_bias;       /* nullable                                       */
    int32_t bias_axis;           /* 0: bias[col], 1: bias[row]                     */
    const int32_t *d_res;        /* nullable int32 residual [rows][ld_res]         */
    int64_t ld_res;              /* elements                                       */
    const uint8_t *d_res_codes;  /* nullable packed residual codes [rows][ld_res_codes] */
    int64_t ld_res_codes;        /* bytes                                          */
    int32_t res_mult;
    int32_t res_levels[4];
} dg_requant;

/* Standalone requant: d_acc [rows][ld_acc] int32 -> d_out packed codes
 * [rows][ld_out] (4 consecutive columns per byte, LSB first; cols % 4 == 0
 * not required, tail codes are 0). */
DG_API dg_status dg_requantize(const int32_t *d_acc, int64_t rows, int64_t cols, int64_t ld_acc,
                        const dg_requant *rq, uint8_t *d_out, int64_t ld_out, void *stream);

/* ---------------------------------------------------------------------------
 * S5/S6/S7/S8 — LUT GEMM (Alg. 1; §3.1):
 *      C[m][n] = sum_{k<K} lut.entries[(W[m][k] << 2) | A[k][n]]     (int32, exact)
 * d_w [M][ldw], d_at [N][lda] packed (K-major, see above).
 * Output: rq == NULL -> int32 C at d_c[m*ldc + n];
 *         rq != NULL -> requantised codes (S7 fused), packed 4 columns (n) per
 *                       byte: d_c is uint8 [M][ldc bytes].
 * variant: 0 auto, 1 cc (CUDA-core PRMT lookups, any table),
 *          2 tc (tcgen05 kind::i8, A operand unpacked into tensor memory): product tables with
 *            int8 levels use d_ws for the int8 expansion of At; NON-product tables with every
 *            |entry| <= 127 run the one-hot K' = 4K form (see dg_lut_gemm_onehot) with both
 *            expanded operands in d_ws; others DG_ERR_UNSUPPORTED;
 *            dg_lut_gemm_workspace_size(M, N, K) bytes cover either form,
 *          3 tc_ss (earlier tcgen05 variant: both operands unpacked to shared memory).
 * auto = tc where it applies, else cc (non-product tables with |entry| > 127).
 * DG_ERR_OVERFLOW if K * max|entry| >= 2^31.  With rq, |acc + bias| < 2^30 is
 * required for the fused fast path's int32 threshold compare (else exact int64). */
DG_API size_t dg_lut_gemm_workspace_size(int64_t M, int64_t N, int64_t K);
DG_API dg_status dg_lut_gemm(const uint8_t *d_w, int64_t ldw, const uint8_t *d_at, int64_t lda, int64_t M,
                      int64_t N, int64_t K, const dg_lut *lut, void *d_c, int64_t ldc,
                      const dg_requant *rq, void *d_ws, size_t ws_bytes, int32_t variant, void *stream);

/* Offline operand expansion for the tensor-core path: packed codes [rows][ld] ->
 * int8 levels [rows][ld_out] (ld_out >= dg_expand_ld(K), a multiple of 128), with
 * levels[code] in the byte order documented in csrc/unpack.cuh (the 16 codes of a
 * 32-bit word as 0,2,..,14,1,3,..,15; the same order the kernel gives the other
 * operand) and 0 for every k >= K.  Like the paper's offline weight packing and
 * reordering this is done once per weight tensor. */
DG_API int64_t dg_expand_ld(int64_t K);
DG_API dg_status dg_expand_operand(const uint8_t *d_packed, int64_t rows, int64_t K, int64_t ld,
                            const int32_t levels[4], int8_t *d_out, int64_t ld_out, void *stream);

/* Non-product tables on the int8 tensor cores (the one-hot K' = 4K form).
 * Any table splits over the weight code, T[(w<<2)|a] = sum_i [w == i] * T[(i<<2)|a] (Alg. 1's
 * lookup), so C = P' . Q'^T over K' = 4K with
 *      P'[m][4k+i] = [W[m][k] == i]   (packed 2-bit one-hot codes: byte k = 1 << (2 W[m][k]))
 *      Q'[n][4k+i] = T[(i<<2) | A[k][n]]   (int8, in the tensor-core operand order of
 *                                           dg_expand_operand; 0 for k >= K)
 * an exact int8 dot product.  dg_expand_onehot: packed weights [rows][ld] -> [rows][ld_out]
 * (ld_out >= dg_onehot_ld(K) = roundup(K, 16), a multiple of 16); dg_expand_tcols: packed
 * activations [rows][ld] -> int8 [rows][ld_out] (ld_out >= dg_tcols_ld(K) = dg_expand_ld(4K), a
 * multiple of 128, 128-byte aligned); both once per operand.  dg_lut_gemm_onehot: output and
 * rq as dg_lut_gemm.  Requires every |entry| <= 127 (else DG_ERR_UNSUPPORTED); d_atc must have
 * been built from the same table.  4x the MMA work of the product-table path, any table.     */
DG_API int64_t dg_onehot_ld(int64_t K);
DG_API int64_t dg_tcols_ld(int64_t K);
DG_API dg_status dg_expand_onehot(const uint8_t *d_w, int64_t rows, int64_t K, int64_t ld, uint8_t *d_out,
                                  int64_t ld_out, void *stream);
DG_API dg_status dg_expand_tcols(const uint8_t *d_at, int64_t rows, int64_t K, int64_t ld, const dg_lut *lut,
                                 int8_t *d_out, int64_t ld_out, void *stream);
DG_API dg_status dg_lut_gemm_onehot(const uint8_t *d_w1h, int64_t ldw1h, const int8_t *d_atc, int64_t ldatc,
                                    int64_t M, int64_t N, int64_t K, const dg_lut *lut, void *d_c, int64_t ldc,
                                    const dg_requant *rq, void *stream);

/* 4-bit operands (Table 2: b-bit LUTs with 2^(2b) entries) on the
 * 2-bit tensor-core path, for product tables with IDENTITY activation levels (al[a] = a, a in
 * 0..15: unsigned ReLU-style codes) and any 16 int8 weight levels with |4 wl| <= 127:
 *      C[m][n] = sum_{k<K} wl[W[m][k]] * A[k][n]     (= sum_k T[(W << 4) | A], T = wl x {0..15})
 * A 4-bit code is the two 2-bit digits a = a_l + 4 a_h, and a packed 4-bit row (code k in nibble
 * k&1 of byte k>>1, low nibble first: the same bytes as the 2-bit packing of the digit sequence
 * a_l0, a_h0, a_l1, ...: dg_pack_codes4 writes it) is a packed 2-bit row of
 * K' = 2K digits; the weights become Q'[2k] = wl[w_k], Q'[2k+1] = 4 wl[w_k] (dg_expand_digits4:
 * packed 4-bit weights [rows][ld] -> int8 [rows][ld_out], ld_out >= dg_expand_ld(2K), a multiple
 * of 128, 128-byte aligned; DG_ERR_RANGE if some |4 wl| > 127).  Out-of-image conv taps read
 * code 0.
 * dg_lut_gemm4_prepared: d_at4 [N][lda] packed 4-bit activations, d_w8 = dg_expand_digits4(W);
 *      output in the activation-major orientation Ct[n][m] (the NHWC convention of the conv
 *      calls): int32 [N][ldct], or with rq the requantised codes of C^T packed 4 m per byte.
 * dg_lut_conv2d4_prepared: p->C = the number of 4-bit channels (x: [B][H][W][C/2] bytes),
 *      d_w8 = dg_expand_digits4 of the packed 4-bit weights [Cout][kh*kw*C] (K order r, s, c);
 *      p->pad_code must be 0; otherwise as dg_lut_conv2d_prepared.                            */
/* Packs 4-bit codes (one per byte, [rows][ld_codes]; values > 15 are masked with &15 and counted
 * into *d_err_count when non-NULL) into packed 4-bit rows [rows][ld]: code k in nibble k&1 of
 * byte k>>1, low nibble first, zero beyond K; ld % 16 == 0, ld >= ceil(K/2), d_packed 16-byte
 * aligned (DG_ERR_INVALID_ARG otherwise). */
DG_API dg_status dg_pack_codes4(const uint8_t *d_codes, int64_t rows, int64_t K, int64_t ld_codes, uint8_t *d_packed,
                                int64_t ld, int32_t *d_err_count, void *stream);
DG_API dg_status dg_expand_digits4(const uint8_t *d_w4, int64_t rows, int64_t K, int64_t ld, const int32_t levels[16],
                                   int8_t *d_out, int64_t ld_out, void *stream);
DG_API dg_status dg_lut_gemm4_prepared(const uint8_t *d_at4, int64_t lda, const int8_t *d_w8, int64_t ld8, int64_t N,
                                       int64_t M, int64_t K, const int32_t levels[16], void *d_ct, int64_t ldct,
                                       const dg_requant *rq, void *stream);

/* FLOAT-valued tables (§5.3: "The LUT can store either integer or floating-point values";
 * e.g. the products of a non-uniform quantiser's levels):
 *      C[m][n] = sum_{k<K} table[(W[m][k] << 2) | A[k][n]]          (fp32 output C [M][ldc])
 * on the int8 tensor cores: the table is written in fixed point, Ti = rne(table * 2^s) with the
 * largest s keeping max|Ti| <= Q = 127 (2^16 + 2^8 + 1), split into three balanced int8 digits
 * Ti = d2 2^16 + d1 2^8 + d0; the three digit LUT sums are exact int8 dot products in the one-hot
 * form (dg_lut_gemm_onehot), and (acc2 2^16 + acc1 2^8 + acc0) 2^-s is formed exactly in fp64
 * before one rounding to fp32.  Error bound (reading Q24), tested against the fp64 oracle:
 *      |C - sum_k table[...]| <= K max|table| / Q + 2^-24 |sum_k table[...]|
 * (exact up to the final rounding when every entry is a multiple of 2^-s).  d_ws:
 * dg_lut_gemm_f32_workspace_size(M, N, K) bytes.  DG_ERR_RANGE for a non-finite entry,
 * DG_ERR_OVERFLOW for K >= 2^22.  dg_float_table_fixed (host) returns s and the digits
 * (digits[16 j + e] = d_j of entry e) for inspection.                                           */
DG_API dg_status dg_float_table_fixed(const float table[16], int32_t digits[48], int32_t *shift);
DG_API size_t dg_lut_gemm_f32_workspace_size(int64_t M, int64_t N, int64_t K);
DG_API dg_status dg_lut_gemm_f32(const uint8_t *d_w, int64_t ldw, const uint8_t *d_at, int64_t lda, int64_t M, int64_t N,
                                 int64_t K, const float table[16], float *d_c, int64_t ldc, void *d_ws, size_t ws_bytes,
                                 void *stream);

/* General 4-bit tables (Table 2: 4-bit codes, an 8-bit index (w << 4) | a into a
 * 256-entry table; 3-bit tables are 4-bit tables over codes 0..7): any int8 table (|entry| <= 127,
 * e.g. non-affine activation levels or non-product entries) in the one-hot form over the 16
 * weight codes, K' = 16K, on the int8 tensor cores:
 *      C[m][n] = sum_{k<K} table[(W[m][k] << 4) | A[k][n]]
 * dg_expand_onehot4: packed 4-bit weights [rows][ld] (code k in nibble k&1 of byte k>>1) ->
 *   packed 2-bit one-hot codes [rows][ld_out >= dg_onehot4_ld(K)] (the word 1 << (2 code) per code);
 * dg_expand_tcols4: packed 4-bit activations -> int8 [rows][ld_out >= dg_tcols4_ld(K)] (128-byte
 *   aligned) of table[(i << 4) | a] at k' = 16k + i in the tensor-core operand order;
 * dg_lut_gemm4_onehot: output and rq as dg_lut_gemm.  DG_ERR_UNSUPPORTED if some |entry| > 127.  */
DG_API int64_t dg_onehot4_ld(int64_t K);
DG_API int64_t dg_tcols4_ld(int64_t K);
DG_API dg_status dg_expand_onehot4(const uint8_t *d_w4, int64_t rows, int64_t K, int64_t ld, uint8_t *d_out,
                                   int64_t ld_out, void *stream);
DG_API dg_status dg_expand_tcols4(const uint8_t *d_at4, int64_t rows, int64_t K, int64_t ld, const int32_t table[256],
                                  int8_t *d_out, int64_t ld_out, void *stream);
DG_API dg_status dg_lut_gemm4_onehot(const uint8_t *d_w1h, int64_t ldw1h, const int8_t *d_atc, int64_t ldatc, int64_t M,
                                     int64_t N, int64_t K, const int32_t table[256], void *d_c, int64_t ldc,
                                     const dg_requant *rq, void *stream);

/* Block-scaled FP4 tensor-core path (tcgen05 kind::mxf4, e2m1 x e2m1):
 *      C[m][n] = sum_{k<K} lut.entries[(W[m][k] << 2) | A[k][n]]     (int32, exact)
 * for product tables whose activation levels are lut->al = {0, 1, 2, 3} (the activation code is
 * then the e2m1 encoding of al/2, so the kernel unpacks it with two nibble masks per 16 codes) and
 * whose weight levels v have v/2 in e2m1, i.e. v in {0, +-1, +-2, +-3, +-4, +-6, +-8, +-12}
 * (BJ configs 1-4: wl = {-2, -1, 0, 1}).  The fp32 tensor-core sums are integers below 2^22 and
 * exact (tools/fp4_test.cu); DG_ERR_OVERFLOW if K * max|entry| >= 2^22.
 * dg_expand_operand_f4: packed weights [rows][ld] -> e2m1 nibbles of level/2 [rows][ld_out]
 * (ld_out >= dg_expand_f4_ld(K) = roundup(K, 256) / 2, a multiple of 128; 0 for k >= K), done
 * once per weight tensor.  DG_ERR_UNSUPPORTED if a level is not representable.
 * dg_lut_gemm_f4: d_w4 [M][ld4] (expanded weights, 16-byte aligned), d_at [N][lda] packed
 * activations (K-major, lda % 16 == 0), int32 C [M][ldc] (ldc >= N), no requant.
 * DG_ERR_UNSUPPORTED if the table does not qualify (use dg_lut_gemm / _prepared).          */
DG_API int64_t dg_expand_f4_ld(int64_t K);
DG_API dg_status dg_expand_operand_f4(const uint8_t *d_packed, int64_t rows, int64_t K, int64_t ld,
                                      const int32_t levels[4], uint8_t *d_out, int64_t ld_out, void *stream);
DG_API dg_status dg_lut_gemm_f4(const uint8_t *d_w4, int64_t ld4, const uint8_t *d_at, int64_t lda, int64_t M,
                                int64_t N, int64_t K, const dg_lut *lut, int32_t *d_c, int64_t ldc, void *stream);

/* Fused LUT GEMM + all-gather (config 5's exchange step): computes this
 * rank's row block exactly as dg_lut_gemm_prepared with int32 output and no requant,
 * and the epilogue stores every output tile to d_c AND to each of the npeers (<= 7)
 * extra destinations d_c_peers[i] (host array of device pointers: the other ranks'
 * C buffers mapped peer-to-peer, e.g. CUDA IPC / symmetric memory), all with the
 * same row pitch ldc and already offset to this rank's first row.  Where the instance
 * stages int32 tiles for the TMA store, each 32 x 32 chunk leaves the staging buffer once
 * per destination as one bulk tensor store (whole boxes over NVLink, not per-lane stores).  The exchange thus
 * overlaps the math tile by tile instead of following it as a separate collective.
 * Every destination must have the 16-byte alignment of d_c.  The caller orders
 * completion before peers read (e.g. a barrier on the same stream after the call);
 * the kernel fences system-wide before it exits.  DG_ERR_UNSUPPORTED if npeers > 7. */
DG_API dg_status dg_lut_gemm_prepared_allgather(const uint8_t *d_w, int64_t ldw, const int8_t *d_at8, int64_t ld8,
                                         int64_t M, int64_t N, int64_t K, const dg_lut *lut, int32_t *d_c,
                                         int64_t ldc, int32_t *const *d_c_peers, int32_t npeers, void *stream);

/* LUT GEMM with a prepared second operand (tc path only):
 *      C[m][n] = sum_{k<K} lut.entries[(W[m][k] << 2) | A[k][n]]
 * d_w packed [M][ldw]; d_at8 = dg_expand_operand(At, levels = lut->al) [N][ld8].
 * Requires lut->is_product with int8 levels.  Output as dg_lut_gemm.       */
DG_API dg_status dg_lut_gemm_prepared(const uint8_t *d_w, int64_t ldw, const int8_t *d_at8, int64_t ld8,
                               int64_t M, int64_t N, int64_t K, const dg_lut *lut, void *d_c, int64_t ldc,
                               const dg_requant *rq, void *stream);

/* ---------------------------------------------------------------------------
 * Convolution over packed NHWC codes = im2col (S3) + LUT GEMM (S5) + fused
 * requant (S7), output NHWC (conv layers are run as (M,N,K) GEMMs).
 * On the tc path, convs whose C/4 is a power of two >= 16 skip the im2col matrix
 * (implicit GEMM: the kernel gathers each output pixel's taps):
 *      out[b][ho][wo][co] = sum_{r,s,c} T[(w[co][r][s][c] << 2) | x(b, ho*st-pad+r, wo*st-pad+s, c)]
 * d_x: [B][H][W][C/4] packed; d_w: [Cout][ldw] packed rows of K = kh*kw*C codes
 * in (r,s,c) order.  Output: rq == NULL -> int32 [B*Ho*Wo][Cout];
 * rq != NULL -> packed codes [B*Ho*Wo][Cout/4] (Cout % 4 == 0), the next
 * layer's NHWC input.  Residuals / bias in rq are indexed [pixel][cout].    */
typedef struct {
    int32_t B, H, W, C, Cout, kh, kw, stride, pad;
    int32_t pad_code;
    int64_t ldw;
} dg_conv_params;

DG_API size_t dg_lut_conv2d_workspace_size(const dg_conv_params *p);
DG_API dg_status dg_lut_conv2d(const uint8_t *d_x, const uint8_t *d_w, const dg_lut *lut,
                        const dg_conv_params *p, const dg_requant *rq, void *d_out, void *d_ws,
                        size_t ws_bytes, int32_t variant, void *stream);

/* Convolution with offline-expanded weights (tc path only): d_w8 = dg_expand_operand(weights,
 * levels = lut->wl) [Cout][ld8].  1x1/stride-1 convs read x directly; convs whose C/4 is a
 * power of two >= 16 run as an implicit GEMM (the kernel gathers each output pixel's taps from
 * x; no im2col matrix); others use dg_im2col into d_ws (dg_lut_conv2d_workspace_size bytes). */
DG_API dg_status dg_lut_conv2d_prepared(const uint8_t *d_x, const int8_t *d_w8, int64_t ld8, const dg_lut *lut,
                                 const dg_conv_params *p, const dg_requant *rq, void *d_out, void *d_ws,
                                 size_t ws_bytes, void *stream);

/* Convolution on the block-scaled FP4 tensor-core path (tcgen05 kind::mxf4):
 * the same result as dg_lut_conv2d_prepared for product tables whose activation levels are
 * lut->al = {0, 1, 2, 3} and whose weight levels v have v/2 in e2m1 (see dg_lut_gemm_f4), with
 * K * max|entry| < 2^22 (else DG_ERR_OVERFLOW).  d_w4 = dg_expand_operand_f4(weights [Cout][K],
 * levels = lut->wl) [Cout][ld4], K order (r, s, c).  The activation codes are unpacked on chip into
 * e2m1 nibbles; 1x1 / stride-1 convs read x directly, others gather their taps (C/4 a power of
 * two >= 16).  Output as dg_lut_conv2d_prepared.  DG_ERR_UNSUPPORTED (use the int8 path) for:
 * residuals in rq, bias per row, requant parameters without a 16-bit form, other channel counts,
 * Cout > 2048.  The expanded weights / bias are read before the programmatic-dependent-launch wait
 * only under the "early_weights" option.                                                        */
DG_API dg_status dg_lut_conv2d_f4_prepared(const uint8_t *d_x, const uint8_t *d_w4, int64_t ld4, const dg_lut *lut,
                                           const dg_conv_params *p, const dg_requant *rq, void *d_out, void *stream);

/* 4-bit convolution (see dg_lut_gemm4_prepared above for the digit form and its requirements). */
DG_API dg_status dg_lut_conv2d4_prepared(const uint8_t *d_x4, const int8_t *d_w8, int64_t ld8,
                                         const int32_t levels[16], const dg_conv_params *p,
                                         const dg_requant *rq, void *d_out, void *d_ws, size_t ws_bytes,
                                         void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DG_H_ */
