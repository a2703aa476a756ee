// pack.cu — S1/S2/S3/S7 streaming kernels: pack, unpack, Eq. 1 quantise+pack,
// packed im2col, standalone requant.  All HBM-bound: 128-bit loads/stores where the
// layout allows, grid-stride loops sized to a multiple of the SM count.
//
// Packed format: dg.h (Fig. 1a caption, §3.1; reading Q20).
#include "common.cuh"

namespace dg {
namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t work, int per_block = kThreads) {
    int64_t b = (work + per_block - 1) / per_block;
    int64_t cap = (int64_t)num_sms() * 8;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

// Pack 4 codes (one per byte of w) into one byte: code j -> bits 2j (shift/OR).
DG_DEV uint32_t pack4(uint32_t w) {
    w &= 0x03030303u;
    return (w | (w >> 6) | (w >> 12) | (w >> 18)) & 0xFFu;
}

// ---- S1/S2: pack one-code-per-byte rows into the packed format.
// One thread per output 16-byte chunk (64 codes).
__global__ void pack_kernel(const uint8_t *__restrict__ codes, int64_t rows, int64_t K,
                            int64_t ld_codes, uint8_t *__restrict__ packed, int64_t ld,
                            int32_t *__restrict__ err) {
    const int64_t chunks_per_row = ld / 16;
    const int64_t total = rows * chunks_per_row;
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / chunks_per_row;
        const int64_t ch = i - r * chunks_per_row;
        const int64_t k0 = ch * 64;
        const uint8_t *src = codes + r * ld_codes;
        uint32_t out[4] = {0, 0, 0, 0};
        if (k0 + 64 <= K && (((uintptr_t)(src + k0)) & 15) == 0) {
            const uint4 *s4 = reinterpret_cast<const uint4 *>(src + k0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint4 v = __ldg(s4 + q);
                uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    // count bytes holding a value > 3 (any of bits 2..7 set)
                    uint32_t hi = w[j] & 0xFCFCFCFCu;
                    hi = ((hi >> 2) | (hi >> 3) | (hi >> 4) | (hi >> 5) | (hi >> 6) | (hi >> 7)) &
                         0x01010101u;
                    bad += __popc(hi);
                    out[q] |= pack4(w[j]) << (8 * j);
                }
            }
        } else {
            for (int64_t k = k0; k < k0 + 64 && k < K; ++k) {
                uint32_t c = src[k];
                if (c > 3) bad += 1;
                out[(k - k0) >> 4] |= (c & 3u) << (2 * ((k - k0) & 15));
            }
        }
        *reinterpret_cast<uint4 *>(packed + r * ld + ch * 16) = make_uint4(out[0], out[1], out[2], out[3]);
    }
    if (err && bad) atomicAdd(err, bad);
}

// ---- 4-bit codes (Table 2): one code per byte -> nibble k&1 of byte k>>1, low nibble
// first, zero beyond K.  One thread per output 16-byte chunk (32 codes).
__global__ void pack4_kernel(const uint8_t *__restrict__ codes, int64_t rows, int64_t K, int64_t ld_codes,
                             uint8_t *__restrict__ packed, int64_t ld, int32_t *__restrict__ err) {
    const int64_t chunks_per_row = ld / 16;
    const int64_t total = rows * chunks_per_row;
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / chunks_per_row;
        const int64_t k0 = (i - r * chunks_per_row) * 32;
        const uint8_t *src = codes + r * ld_codes;
        uint32_t out[4] = {0, 0, 0, 0};
        for (int64_t k = k0; k < k0 + 32 && k < K; ++k) {
            const uint32_t c = src[k];
            if (c > 15) bad += 1;
            out[(k - k0) >> 3] |= (c & 15u) << (4 * ((k - k0) & 7));
        }
        *reinterpret_cast<uint4 *>(packed + r * ld + (k0 >> 1)) = make_uint4(out[0], out[1], out[2], out[3]);
    }
    if (err && bad) atomicAdd(err, bad);
}

__global__ void unpack_kernel(const uint8_t *__restrict__ packed, int64_t rows, int64_t K, int64_t ld,
                              uint8_t *__restrict__ codes) {
    const int64_t total = rows * K;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / K, k = i - r * K;
        codes[i] = (packed[r * ld + (k >> 2)] >> (2 * (k & 3))) & 3;
    }
}

// ---- S2: Eq. 1 quantise + pack.  One thread per output byte (4 codes).
__global__ void quantize_pack_kernel(const float *__restrict__ x, int64_t rows, int64_t K, float s,
                                     float z, int32_t qmin, int32_t qmax, uint8_t *__restrict__ packed,
                                     int64_t ld) {
    const int64_t total = rows * ld;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / ld, byte = i - r * ld;
        uint32_t out = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t k = byte * 4 + j;
            if (k < K) {
                float t = roundf(__fmaf_rn(s, x[r * K + k], z));  // roundf: half away from zero
                int32_t q = (t < (float)qmin) ? qmin : ((t > (float)qmax) ? qmax : (int32_t)t);
                out |= (uint32_t)(q - qmin) << (2 * j);
            }
        }
        packed[i] = (uint8_t)out;
    }
}

// ---- S3: packed im2col.  Each output row = kh*kw taps of C/4 bytes, then zeros to ld.
// Block = (VPR vectors of V bytes per row) x (rows); 32-bit index math; the (b, ho, wo)
// decomposition is done once per row.  V = 16 when C/4 % 16 == 0, 4 when % 4 == 0, else 1.
template <int V>
__global__ void __launch_bounds__(256) im2col_kernel(const uint8_t *__restrict__ x, int32_t H, int32_t W, int32_t Cb,
                                                     int32_t kw, int32_t stride, int32_t pad, uint32_t pad_byte,
                                                     int32_t Ho, int32_t Wo, int32_t rows, int32_t kb,
                                                     uint8_t *__restrict__ cols, int32_t ld) {
    const uint32_t vpr = (uint32_t)(ld / V);
    const uint32_t total = (uint32_t)rows * vpr;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const uint32_t row = i / vpr;
        const int32_t byte = (int32_t)(i - row * vpr) * V;
        uint8_t *dst = cols + (int64_t)row * ld + byte;
        if (byte >= kb) {  // K tail: zero codes (dg.h contract)
            if constexpr (V == 16) *reinterpret_cast<uint4 *>(dst) = make_uint4(0, 0, 0, 0);
            else if constexpr (V == 4) *reinterpret_cast<uint32_t *>(dst) = 0;
            else *dst = 0;
            continue;
        }
        const uint32_t t = row / (uint32_t)Wo;
        const int32_t wo = (int32_t)(row - t * (uint32_t)Wo);
        const uint32_t b = t / (uint32_t)Ho;
        const int32_t ho = (int32_t)(t - b * (uint32_t)Ho);
        const int32_t tap = byte / Cb;
        const int32_t cb = byte - tap * Cb;
        const int32_t r = tap / kw, s = tap - r * kw;
        const int32_t hi = ho * stride - pad + r, wi = wo * stride - pad + s;
        const bool in = (uint32_t)hi < (uint32_t)H && (uint32_t)wi < (uint32_t)W;
        const uint8_t *src = x + (((int64_t)b * H + hi) * W + wi) * Cb + cb;
        if constexpr (V == 16) {
            const uint4 val = in ? __ldg(reinterpret_cast<const uint4 *>(src)) : make_uint4(pad_byte, pad_byte, pad_byte, pad_byte);
            *reinterpret_cast<uint4 *>(dst) = val;
        } else if constexpr (V == 4) {
            *reinterpret_cast<uint32_t *>(dst) = in ? __ldg(reinterpret_cast<const uint32_t *>(src)) : pad_byte;
        } else {
            *dst = in ? __ldg(src) : (uint8_t)pad_byte;
        }
    }
}

// Narrow pixels (C/4 % 4 != 0, e.g. VGG conv1_1's C = 3 -> 4: one packed byte per pixel), short rows
// (ld <= 64 bytes): one thread per output ROW forms (b, ho, wo) once and assembles the row's
// kh*kw*Cb bytes in registers, then writes it with 16-byte stores (the byte-per-thread form above
// did two divisions and a byte store per output byte: 260 us for VGG conv1_1 at batch 64).
template <int KH, int KW, int CB>   // 0: runtime (kh, kw, Cb)
__global__ void __launch_bounds__(256) im2col_rows_kernel(const uint8_t *__restrict__ x, int32_t H, int32_t W,
                                                          int32_t Cb_, int32_t kh_, int32_t kw_, int32_t stride,
                                                          int32_t pad, uint32_t pad_byte, int32_t Ho, int32_t Wo,
                                                          int32_t rows, uint8_t *__restrict__ cols, int32_t ld) {
    const int32_t kh = KH ? KH : kh_, kw = KW ? KW : kw_, Cb = CB ? CB : Cb_;
    (void)kh;
    (void)kw;
    for (int32_t row = blockIdx.x * blockDim.x + threadIdx.x; row < rows; row += gridDim.x * blockDim.x) {
        const int32_t t = row / Wo, wo = row - t * Wo;
        const int32_t b = t / Ho, ho = t - b * Ho;
        uint32_t w[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) w[j] = 0;
        const uint8_t *img = x + (int64_t)b * H * W * Cb;
        if constexpr (KH && KW && CB) {   // every byte index a compile-time constant
#pragma unroll
            for (int32_t r = 0; r < KH; ++r) {
                const int32_t hi = ho * stride - pad + r;
#pragma unroll
                for (int32_t s = 0; s < KW; ++s) {
                    const int32_t wi = wo * stride - pad + s;
                    const bool in = (uint32_t)hi < (uint32_t)H && (uint32_t)wi < (uint32_t)W;
                    const uint8_t *src = img + (hi * W + wi) * CB;
#pragma unroll
                    for (int32_t c = 0; c < CB; ++c) {
                        const int32_t idx = (r * KW + s) * CB + c;
                        w[idx >> 2] |= (in ? (uint32_t)__ldg(src + c) : pad_byte) << (8 * (idx & 3));
                    }
                }
            }
        } else {
            int32_t idx = 0;
#pragma unroll 1
            for (int32_t r = 0; r < kh; ++r) {
                const int32_t hi = ho * stride - pad + r;
#pragma unroll 1
                for (int32_t s = 0; s < kw; ++s) {
                    const int32_t wi = wo * stride - pad + s;
                    const bool in = (uint32_t)hi < (uint32_t)H && (uint32_t)wi < (uint32_t)W;
                    const uint8_t *src = img + (hi * W + wi) * Cb;
#pragma unroll 1
                    for (int32_t c = 0; c < Cb; ++c, ++idx) {
                        const uint32_t v = in ? (uint32_t)__ldg(src + c) : pad_byte;
#pragma unroll
                        for (int j = 0; j < 16; ++j)   // (register-resident: word idx >> 2 by compare)
                            if (j == (idx >> 2)) w[j] |= v << (8 * (idx & 3));
                    }
                }
            }
        }
        uint4 *dst = reinterpret_cast<uint4 *>(cols + (int64_t)row * ld);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (16 * j < ld) dst[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
    }
}

template <int V>
void launch_im2col(const uint8_t *x, int32_t B, int32_t H, int32_t W, int32_t Cb, int32_t kh, int32_t kw, int32_t stride,
                   int32_t pad, uint32_t pad_byte, int32_t Ho, int32_t Wo, uint8_t *cols, int64_t ld, cudaStream_t st) {
    const int32_t rows = B * Ho * Wo;
    const int64_t total = (int64_t)rows * (ld / V);
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = (int64_t)num_sms() * 16;
    if (blocks > cap) blocks = cap;
    im2col_kernel<V><<<(int)blocks, 256, 0, st>>>(x, H, W, Cb, kw, stride, pad, pad_byte, Ho, Wo, rows, kh * kw * Cb,
                                                  cols, (int32_t)ld);
}

// ---- S7 standalone: one thread per output byte (4 columns).
__global__ void requant_kernel(const int32_t *__restrict__ acc, int64_t rows, int64_t cols,
                               int64_t ld_acc, const __grid_constant__ RequantArgs q, uint8_t *__restrict__ out,
                               int64_t ld_out) {
    const int64_t bytes_per_row = (cols + 3) / 4;
    const int64_t total = rows * bytes_per_row;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / bytes_per_row, b = i - r * bytes_per_row;
        uint32_t o = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t c = b * 4 + j;
            if (c < cols) o |= requant_one(q, acc[r * ld_acc + c], r, c) << (2 * j);
        }
        out[r * ld_out + b] = (uint8_t)o;
    }
}

}  // namespace
}  // namespace dg

using namespace dg;

extern "C" {

int64_t dg_packed_ld(int64_t K) {
    if (K <= 0) return 0;
    int64_t b = (K + 3) / 4;
    return (b + 15) / 16 * 16;
}

static dg_status pack_common(const uint8_t *d_codes, int64_t rows, int64_t K, int64_t ld_codes,
                             uint8_t *d_packed, int64_t ld, int32_t *d_err, void *stream) {
    if (!d_codes || !d_packed) return DG_ERR_INVALID_ARG;
    if (rows < 0 || K <= 0 || ld_codes < K) return DG_ERR_SHAPE;
    if (ld % 16 != 0 || ld * 4 < K || ((uintptr_t)d_packed & 15)) return DG_ERR_INVALID_ARG;
    if (rows == 0) return DG_OK;
    const int64_t work = rows * (ld / 16);
    pack_kernel<<<grid_for(work), kThreads, 0, (cudaStream_t)stream>>>(d_codes, rows, K, ld_codes,
                                                                       d_packed, ld, d_err);
    return launch_status();
}

dg_status dg_pack_codes(const uint8_t *d_codes, int64_t rows, int64_t K, int64_t ld_codes,
                        uint8_t *d_packed, int64_t ld, int32_t *d_err_count, void *stream) {
    return pack_common(d_codes, rows, K, ld_codes, d_packed, ld, d_err_count, stream);
}

dg_status dg_pack_weights(const uint8_t *d_codes, int64_t rows, int64_t K, int64_t ld_codes,
                          uint8_t *d_packed, int64_t ld, int32_t *d_err_count, void *stream) {
    return pack_common(d_codes, rows, K, ld_codes, d_packed, ld, d_err_count, stream);
}

dg_status dg_pack_codes4(const uint8_t *d_codes, int64_t rows, int64_t K, int64_t ld_codes, uint8_t *d_packed, int64_t ld,
                         int32_t *d_err_count, void *stream) {
    if (!d_codes || !d_packed) return DG_ERR_INVALID_ARG;
    if (rows < 0 || K <= 0 || ld_codes < K) return DG_ERR_SHAPE;
    if (ld % 16 != 0 || ld * 2 < K || ((uintptr_t)d_packed & 15)) return DG_ERR_INVALID_ARG;
    if (rows == 0) return DG_OK;
    pack4_kernel<<<grid_for(rows * (ld / 16)), kThreads, 0, (cudaStream_t)stream>>>(d_codes, rows, K, ld_codes, d_packed,
                                                                                  ld, d_err_count);
    return launch_status();
}

dg_status dg_unpack_codes(const uint8_t *d_packed, int64_t rows, int64_t K, int64_t ld,
                          uint8_t *d_codes, void *stream) {
    if (!d_packed || !d_codes) return DG_ERR_INVALID_ARG;
    if (rows < 0 || K <= 0 || ld * 4 < K) return DG_ERR_SHAPE;
    if (rows == 0) return DG_OK;
    unpack_kernel<<<grid_for(rows * K), kThreads, 0, (cudaStream_t)stream>>>(d_packed, rows, K, ld, d_codes);
    return launch_status();
}

dg_status dg_quantize_pack_activations(const float *d_x, int64_t rows, int64_t K, float scale,
                                       float zero_point, int32_t qmin, int32_t qmax,
                                       uint8_t *d_packed, int64_t ld, void *stream) {
    if (!d_x || !d_packed) return DG_ERR_INVALID_ARG;
    if (rows < 0 || K <= 0 || ld * 4 < K || ld % 16 != 0) return DG_ERR_SHAPE;
    if (qmax < qmin || qmax - qmin > 3) return DG_ERR_RANGE;
    if (rows == 0) return DG_OK;
    quantize_pack_kernel<<<grid_for(rows * ld), kThreads, 0, (cudaStream_t)stream>>>(
        d_x, rows, K, scale, zero_point, qmin, qmax, d_packed, ld);
    return launch_status();
}

dg_status dg_im2col(const uint8_t *d_x, int32_t B, int32_t H, int32_t W, int32_t C, int32_t kh,
                    int32_t kw, int32_t stride, int32_t pad, uint8_t pad_code, uint8_t *d_cols,
                    int64_t ld, void *stream) {
    if (!d_x || !d_cols) return DG_ERR_INVALID_ARG;
    if (B <= 0 || H <= 0 || W <= 0 || C <= 0 || kh <= 0 || kw <= 0 || stride <= 0 || pad < 0)
        return DG_ERR_SHAPE;
    if (C % 4 != 0 || pad_code > 3) return DG_ERR_RANGE;
    const int32_t Ho = (H + 2 * pad - kh) / stride + 1, Wo = (W + 2 * pad - kw) / stride + 1;
    if (Ho <= 0 || Wo <= 0) return DG_ERR_SHAPE;
    const int32_t Cb = C / 4;
    if (ld % 16 != 0 || ld < (int64_t)kh * kw * Cb || ((uintptr_t)d_cols & 15)) return DG_ERR_INVALID_ARG;
    const uint32_t pb = pad_code | (pad_code << 2) | (pad_code << 4) | (pad_code << 6);
    const int64_t rows = (int64_t)B * Ho * Wo;
    if (rows * (ld / 1) > (int64_t)UINT32_MAX || ld > INT32_MAX / 2) return DG_ERR_SHAPE;
    cudaStream_t st = (cudaStream_t)stream;
    if (Cb % 16 == 0 && ((uintptr_t)d_x & 15) == 0) {
        launch_im2col<16>(d_x, B, H, W, Cb, kh, kw, stride, pad, pb * 0x01010101u, Ho, Wo, d_cols, ld, st);
    } else if (Cb % 4 == 0 && ((uintptr_t)d_x & 3) == 0) {
        launch_im2col<4>(d_x, B, H, W, Cb, kh, kw, stride, pad, pb * 0x01010101u, Ho, Wo, d_cols, ld, st);
    } else if (ld <= 64 && rows <= INT32_MAX && kh <= 8 && kw <= 8 && Cb <= 3 &&
               (int64_t)B * H * W * Cb <= INT32_MAX) {
        int64_t blocks = (rows + 255) / 256;
        if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
        if (kh == 3 && kw == 3 && Cb == 1)   // (VGG / ResNet stems after padding C = 3 to 4)
            im2col_rows_kernel<3, 3, 1><<<(int)blocks, 256, 0, st>>>(d_x, H, W, Cb, kh, kw, stride, pad, pb, Ho, Wo,
                                                                     (int32_t)rows, d_cols, (int32_t)ld);
        else
            im2col_rows_kernel<0, 0, 0><<<(int)blocks, 256, 0, st>>>(d_x, H, W, Cb, kh, kw, stride, pad, pb, Ho, Wo,
                                                                     (int32_t)rows, d_cols, (int32_t)ld);
    } else {
        launch_im2col<1>(d_x, B, H, W, Cb, kh, kw, stride, pad, pb, Ho, Wo, d_cols, ld, st);
    }
    return launch_status();
}

dg_status dg_requantize(const int32_t *d_acc, int64_t rows, int64_t cols, int64_t ld_acc,
                        const dg_requant *rq, uint8_t *d_out, int64_t ld_out, void *stream) {
    if (!d_acc || !rq || !d_out) return DG_ERR_INVALID_ARG;
    if (rows < 0 || cols <= 0 || ld_acc < cols || ld_out * 4 < cols) return DG_ERR_SHAPE;
    if (rq->qmax < rq->qmin || rq->qmax - rq->qmin > 3 || rq->shift < 0 || rq->shift > 62)
        return DG_ERR_RANGE;
    if (rq->d_res_codes)
        for (int i = 0; i < 4; ++i) {
            const int64_t r = (int64_t)rq->res_levels[i] * rq->res_mult;
            if (r > INT32_MAX || r < INT32_MIN) return DG_ERR_RANGE;
        }
    if (rows == 0) return DG_OK;
    RequantArgs a = to_args(rq);
    requant_kernel<<<grid_for(rows * ((cols + 3) / 4)), kThreads, 0, (cudaStream_t)stream>>>(
        d_acc, rows, cols, ld_acc, a, d_out, ld_out);
    return launch_status();
}

}  // extern "C"
