// common.cuh — shared device/host helpers of libdg (the CUDA path).
// Nothing here is shared with oracle/ (the two sides share no code).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dg.h"

#define DG_DEV __device__ __forceinline__

namespace dg {

// Requantisation of one accumulator (S7; dg.h dg_requant; Eq. 1 with s = mult*2^-shift,
// round half away from zero, reading Q5/Q11).  Exact in int64: |v| < 2^32, |mult| < 2^31.
struct RequantArgs {
    int32_t mult, shift, zp, qmin, qmax;
    const int32_t *bias;
    int32_t bias_axis;
    const int32_t *res;
    int64_t ld_res;
    const uint8_t *res_codes;
    int64_t ld_res_codes;
    int32_t res_mult;
    int32_t res_levels[4];
    // Exact threshold form of the requant map (computed on the host by to_args):
    // code(v) = sum_j [v >= thr[j]] (dir > 0)  or  sum_j [v <= thr[j]] (dir < 0).
    int64_t thr[3];
    int32_t dir;
};

DG_DEV int64_t rhaz(int64_t p, int32_t shift) {
    // round half away from zero of p / 2^shift, branch-free on the magnitude
    const int64_t sgn = p >> 63;                       // 0 or -1
    const int64_t mag = (p ^ sgn) - sgn;
    const int64_t half = shift > 0 ? ((int64_t)1 << (shift - 1)) : 0;
    const int64_t r = (mag + half) >> shift;
    return (r ^ sgn) - sgn;
}

DG_DEV int32_t res_level(const RequantArgs &q, uint32_t code) {
    return (code & 2u) ? ((code & 1u) ? q.res_levels[3] : q.res_levels[2])
                       : ((code & 1u) ? q.res_levels[1] : q.res_levels[0]);
}

// v = acc (+ residual + bias already added by the caller) -> code (S7; dg.h dg_requant).
// code(v) = clip(rhaz(v*mult/2^shift) + zp, qmin, qmax) - qmin is monotone in v, so it is
// evaluated exactly as a count of host-precomputed integer thresholds (no 64-bit multiply).
DG_DEV uint32_t requant_value(const RequantArgs &q, int64_t v) {
    if (q.dir > 0)
        return (uint32_t)(v >= q.thr[0]) + (uint32_t)(v >= q.thr[1]) + (uint32_t)(v >= q.thr[2]);
    return (uint32_t)(v <= q.thr[0]) + (uint32_t)(v <= q.thr[1]) + (uint32_t)(v <= q.thr[2]);
}

// Requantisation of one accumulator element (r, c): adds residual and bias, returns the code.
DG_DEV uint32_t requant_one(const RequantArgs &q, int64_t acc, int64_t r, int64_t c) {
    int64_t v = acc;
    if (q.res) v += q.res[r * q.ld_res + c];
    if (q.res_codes) {
        uint32_t b = q.res_codes[r * q.ld_res_codes + (c >> 2)];
        v += (int64_t)res_level(q, (b >> (2 * (c & 3))) & 3u) * q.res_mult;
    }
    if (q.bias) v += q.bias[q.bias_axis == 0 ? c : r];
    return requant_value(q, v);
}

// Requantise 32 consecutive columns [c0, c0+32) of row r (all valid) -> 64 bits of codes,
// 4 columns per byte LSB first.  Vectorised loads of bias / residuals where aligned.
DG_DEV uint2 requant_row32(const RequantArgs &q, const int32_t (&acc)[32], int64_t r, int64_t c0) {
    int64_t v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = acc[j];
    if (q.bias) {
        if (q.bias_axis == 1) {
            const int64_t b = q.bias[r];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += b;
        } else if ((((uintptr_t)(q.bias + c0)) & 15) == 0) {
            const int4 *b4 = reinterpret_cast<const int4 *>(q.bias + c0);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int4 b = __ldg(b4 + j);
                v[4 * j] += b.x; v[4 * j + 1] += b.y; v[4 * j + 2] += b.z; v[4 * j + 3] += b.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += __ldg(q.bias + c0 + j);
        }
    }
    if (q.res) {
        const int32_t *rp = q.res + r * q.ld_res + c0;
        if ((((uintptr_t)rp) & 15) == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int4 b = __ldg(reinterpret_cast<const int4 *>(rp) + j);
                v[4 * j] += b.x; v[4 * j + 1] += b.y; v[4 * j + 2] += b.z; v[4 * j + 3] += b.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] += __ldg(rp + j);
        }
    }
    if (q.res_codes) {
        const uint8_t *cp = q.res_codes + r * q.ld_res_codes + (c0 >> 2);
        uint32_t w[2];
        if ((((uintptr_t)cp) & 7) == 0) {
            const uint2 t = *reinterpret_cast<const uint2 *>(cp);
            w[0] = t.x; w[1] = t.y;
        } else {
            w[0] = cp[0] | (cp[1] << 8) | (cp[2] << 16) | ((uint32_t)cp[3] << 24);
            w[1] = cp[4] | (cp[5] << 8) | (cp[6] << 16) | ((uint32_t)cp[7] << 24);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j)
            v[j] += (int64_t)res_level(q, (w[j >> 4] >> (2 * (j & 15))) & 3u) * q.res_mult;
    }
    uint32_t o0 = 0, o1 = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) o0 |= requant_value(q, v[j]) << (2 * j);
#pragma unroll
    for (int j = 0; j < 16; ++j) o1 |= requant_value(q, v[16 + j]) << (2 * j);
    return make_uint2(o0, o1);
}

// Host: the requant map evaluated exactly (128-bit product), reference for the thresholds.
inline int64_t requant_code_host(const dg_requant *rq, int64_t v) {
    __int128 p = (__int128)v * rq->mult;
    __int128 mag = p < 0 ? -p : p;
    __int128 half = rq->shift > 0 ? ((__int128)1 << (rq->shift - 1)) : 0;
    __int128 r = (mag + half) >> rq->shift;
    __int128 t = (p < 0 ? -r : r) + rq->zp;
    if (t < rq->qmin) t = rq->qmin;
    if (t > rq->qmax) t = rq->qmax;
    return (int64_t)(t - rq->qmin);
}

inline void requant_thresholds(const dg_requant *rq, RequantArgs &a) {
    const int64_t LO = -((int64_t)1 << 40), HI = ((int64_t)1 << 40);   // |acc+res+bias| < 2^34
    const int64_t NEVER = INT64_MAX, ALWAYS = INT64_MIN;
    a.dir = rq->mult >= 0 ? 1 : -1;
    for (int j = 1; j <= 3; ++j) {
        int64_t t;
        if (a.dir > 0) {   // smallest v with code(v) >= j (code non-decreasing)
            if (requant_code_host(rq, HI) < j) t = NEVER;
            else if (requant_code_host(rq, LO) >= j) t = ALWAYS;
            else {
                int64_t lo = LO, hi = HI;          // code(lo) < j <= code(hi)
                while (hi - lo > 1) { int64_t m = lo + (hi - lo) / 2; (requant_code_host(rq, m) >= j ? hi : lo) = m; }
                t = hi;
            }
        } else {           // largest v with code(v) >= j (code non-increasing)
            if (requant_code_host(rq, LO) < j) t = ALWAYS;
            else if (requant_code_host(rq, HI) >= j) t = NEVER;
            else {
                int64_t lo = LO, hi = HI;          // code(lo) >= j > code(hi)
                while (hi - lo > 1) { int64_t m = lo + (hi - lo) / 2; (requant_code_host(rq, m) >= j ? lo : hi) = m; }
                t = lo;
            }
        }
        a.thr[j - 1] = t;
    }
}

inline RequantArgs to_args(const dg_requant *rq) {
    RequantArgs a{};
    a.mult = rq->mult;
    a.shift = rq->shift;
    a.zp = rq->zp;
    a.qmin = rq->qmin;
    a.qmax = rq->qmax;
    a.bias = rq->d_bias;
    a.bias_axis = rq->bias_axis;
    a.res = rq->d_res;
    a.ld_res = rq->ld_res;
    a.res_codes = rq->d_res_codes;
    a.ld_res_codes = rq->ld_res_codes;
    a.res_mult = rq->res_mult;
    for (int i = 0; i < 4; ++i) a.res_levels[i] = rq->res_levels[i];
    requant_thresholds(rq, a);
    return a;
}

// process-wide count of kernels enqueued by the library (dg_kernel_launches)
uint64_t &launch_counter();

// Runtime options (dg_set_option; read on every call, never cached in a static).  Defaults are
// the tuned dispatch; DG_* environment variables set the initial values (ablations).
enum OptId {
    OPT_WIN,            // 3x3 s1 shifted-window kernel: 0 auto, 1 force for C = 64..256, -1 never
    OPT_WIN128,         // C = 128 tile mode of the window kernel (auto): 1 on, 0 off
    OPT_WPAIR,          // window pair mode (2 row blocks per window): 1 on, 0 off
    OPT_ASM,            // short-K wide tiles with A in shared memory: 1 on, 0 off
    OPT_BN256,          // 128x256 tiles for long K: 1 on, 0 off
    OPT_BN256_K,        // minimum K (codes) for the 128x256 tiles
    OPT_KST,            // codes per pipeline stage: 0 auto, 128 force 128
    OPT_BN64_SHORT,     // short K with Cout > 64 on 64-wide tiles: 0 off, 1 on
    OPT_SPLITK,         // split-K for few-tile long-K GEMMs (workspace given): 1 on, 0 off
    OPT_F16,            // 16-bit SIMD requant epilogue: 1 on, 0 off (32-bit thresholds)
    OPT_BRES,           // resident weight tiles when they fit shared memory: 1 on, 0 off
    OPT_PDL,            // programmatic dependent launch of the TS kernel: 1 on, 0 off
    OPT_EARLY_WEIGHTS,  // *_prepared: load resident weights / bias before griddepcontrol.wait (0 off)
    OPT_F4CONV,         // FP4 (kind::mxf4) kernel for qualifying product-table GEMM/conv layers: 0 off, 1 auto
    OPT_EM,             // epilogue mode of the short-K wide kernel: 0 alternate tiles, 1 column split, 2 high priority, 3 both
    OPT_TMA_STORE,      // int32 output tiles through the TMA tensor store where the instance has staging: 1 on, 0 off
    OPT_UNP,            // unpack warps of the 128x256 long-K instance: 8 (default), 12 or 16
    OPT_F4_UNP,         // FP4 conv kernel unpack warps: 0 auto (4 direct, 8 gathered), 4 or 8
    OPT_F4_EPI,         // FP4 conv kernel epilogue warps: 0 auto, 4 or 8
    OPT_F4_BN,          // FP4 conv tile width: 0 auto (256 when 256 | Cout), 128 or 256
    OPT_F4_OMMA,        // FP4 conv kernel: accumulator origin from one MMA per tile (1) or reset stores (0)
    OPT_F4_CT,          // FP4 conv kernel: CTAs per SM for 128-wide tiles (2) or 1 (0 / 1)
    OPT_SKFUSE,         // split-K slices reduced by the GEMM kernel itself after a grid barrier (1) or a second kernel (0, default)
    OPT_F4_WIN,         // FP4 conv kernel: shifted window for direct 3x3 s1 p1 convs over 64 / 128 channels: 2 auto (resident weights), 1 always, 0 off
    OPT_OFFS,           // short-K shared-memory-A instance: per-column requant offsets from one MMA per tile (1), 0 off
    OPT_BMC,            // TS kernel: B stages multicast across 2-CTA clusters where the tile walk allows (1), 0 off (default)
    OPT_F4_WBRES,       // FP4 conv shifted window: weights resident when one column block fits the B ring (1), 0 off
    OPT_F4_I2C,         // FP4 conv: strided 1x1 convs on the direct path through an im2col-mode tensor map (1), 0 gathered
    OPT_F4_W1X1,        // FP4 conv: 1x1 stride-1 convs into 64 / 128 channels as window pairs: 1 over 64 channels, 2 over <= 256, 0 never
    OPT_F4_WPAIR,       // FP4 conv shifted window, 64 / 128-wide resident tiles: one window per two 128-row blocks (1), 0 off
    OPT_COUNT
};
int64_t opt(OptId id);
// tag of the GEMM kernel instance this thread launched last (dg_last_kernel)
void set_last_kernel(const char *tag);
// 16-bit SIMD requant constants (m, c) for thresholds t0 <= t1 <= t2, verified for every x (lut_gemm_ts.cu)
bool f16_params(int64_t t0, int64_t t1, int64_t t2, uint32_t &m_out, uint32_t &c_out);
inline dg_status launch_status(int nlaunched = 1) {
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) __atomic_fetch_add(&launch_counter(), (uint64_t)nlaunched, __ATOMIC_RELAXED);
    return e == cudaSuccess ? DG_OK : DG_ERR_CUDA;
}

inline int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

}  // namespace dg

// Internal (non-ABI) launchers implemented in the .cu files.
namespace dg {
struct CcTable;  // lut_gemm_cc.cu
dg_status lut_gemm_cc(const uint8_t *P, int64_t ldp, const uint8_t *Q, int64_t ldq, int64_t np,
                      int64_t nq, int64_t K, const int32_t Tt[16], void *D, int64_t ldd,
                      const RequantArgs *rq, cudaStream_t st);
dg_status lut_gemm_tc(const uint8_t *P, int64_t ldp, const uint8_t *Q, int64_t ldq, int64_t np,
                      int64_t nq, int64_t K, const int32_t pl[4], const int32_t ql[4], void *D,
                      int64_t ldd, const RequantArgs *rq, cudaStream_t st);
bool tc_available();
int64_t expand_ld(int64_t K);
dg_status expand_operand(const uint8_t *packed, int64_t rows, int64_t K, int64_t ld, const int32_t levels[4],
                         int8_t *out, int64_t ld8, cudaStream_t st);
// implicit-GEMM convolution description for the TS kernel (P = im2col of x, gathered on chip)
int64_t onehot_ld(int64_t K);
int64_t onehot4_ld(int64_t K);
int64_t tcols4_ld(int64_t K);
dg_status expand_onehot4(const uint8_t *w4, int64_t rows, int64_t K, int64_t ld, uint8_t *out, int64_t ld_out,
                         cudaStream_t st);
dg_status expand_tcols4(const uint8_t *a4, int64_t rows, int64_t K, int64_t ld, const int32_t table[256], int8_t *out,
                        int64_t ld_out, cudaStream_t st);
int64_t tcols_ld(int64_t K);
dg_status expand_onehot(const uint8_t *w, int64_t rows, int64_t K, int64_t ld, uint8_t *out, int64_t ld_out,
                        cudaStream_t st);
dg_status expand_tcols(const uint8_t *a, int64_t rows, int64_t K, int64_t ld, const int32_t entries[16], int8_t *out,
                       int64_t ld_out, cudaStream_t st);
dg_status expand_digits4(const uint8_t *w4, int64_t rows, int64_t K, int64_t ld, const int32_t levels[16], int8_t *out,
                         int64_t ld_out, cudaStream_t st);
int64_t expand_f4_ld(int64_t K);
int f4_nibble_half(int32_t v);
dg_status expand_operand_f4(const uint8_t *packed, int64_t rows, int64_t K, int64_t ld, const int32_t levels[4],
                            uint8_t *out, int64_t ld4, cudaStream_t st);
dg_status lut_gemm_f4(const uint8_t *At, int64_t lda, const uint8_t *W4, int64_t ld4, int64_t M, int64_t N, int64_t K,
                      int32_t *C, int64_t ldc, cudaStream_t st);
struct TsConv {
    const uint8_t *x;
    int32_t H, W, Cb, kh, kw, stride, pad, Ho, Wo, pad_code;
};
bool float_table_digits(const float T[16], int32_t digits[3][16], int32_t *s_out);
int64_t lut_gemm_f32_workspace(int64_t M, int64_t N, int64_t K);
dg_status lut_gemm_f32(const uint8_t *W, int64_t ldw, const uint8_t *At, int64_t lda, int64_t M, int64_t N, int64_t K,
                       const float T[16], float *C, int64_t ldc, void *ws, size_t ws_bytes, cudaStream_t st);
dg_status lut_conv_f4(const uint8_t *x, const uint8_t *w4, int64_t ld4, const TsConv &cv, int64_t rows, int64_t cout,
                      int64_t K, int64_t acc_bound, void *out, int64_t ldd, const RequantArgs *rq, cudaStream_t st,
                      bool b_prepared);
dg_status lut_gemm_ts(const uint8_t *P, int64_t ldp, const int8_t *Q8, int64_t ld8, int64_t np, int64_t nq, int64_t K,
                      const int32_t pl[4], const int32_t ql[4], void *D, int64_t ldd, const RequantArgs *rq,
                      cudaStream_t st, const TsConv *cv = nullptr, void *skws = nullptr, size_t skws_bytes = 0,
                      int32_t *const *peers = nullptr, int32_t npeers = 0, bool b_prepared = false);
}  // namespace dg
