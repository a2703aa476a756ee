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
};

DG_DEV int64_t rhaz(int64_t p, int32_t shift) {
    if (shift == 0) return p;
    const int64_t half = (int64_t)1 << (shift - 1);
    return p >= 0 ? ((p + half) >> shift) : -((-p + half) >> shift);
}

// v already includes acc; adds residual and bias of element (r, c) and returns the code.
DG_DEV uint32_t requant_one(const RequantArgs &q, int64_t acc, int64_t r, int64_t c) {
    int64_t v = acc;
    if (q.res) v += q.res[r * q.ld_res + c];
    if (q.res_codes) {
        uint32_t b = q.res_codes[r * q.ld_res_codes + (c >> 2)];
        uint32_t code = (b >> (2 * (c & 3))) & 3u;
        v += (int64_t)q.res_levels[code] * q.res_mult;
    }
    if (q.bias) v += q.bias[q.bias_axis == 0 ? c : r];
    int64_t t = rhaz(v * (int64_t)q.mult, q.shift) + q.zp;
    t = t < q.qmin ? q.qmin : (t > q.qmax ? q.qmax : t);
    return (uint32_t)(t - q.qmin);
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
    return a;
}

inline dg_status launch_status() {
    cudaError_t e = cudaGetLastError();
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
}  // namespace dg
