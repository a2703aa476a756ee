// im2col_test.cu — semantics check of the TMA im2col mode on packed 2-bit NHWC activations
// (uint8 "channels" = C/4 packed bytes), for the implicit-GEMM conv gather.
// For a tile of PPC consecutive output pixels starting at output pixel p0 and a filter tap (r, s),
// one cp.async.bulk.tensor.4d...im2col load should bring the PPC im2col rows' Cb bytes of that tap
// (out-of-image taps zero-filled) into shared memory as [PPC][Cb].  Compared with a CPU im2col for
// several bounding-box corner conventions; prints which one matches.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/im2col_test tools/im2col_test.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../paper_2304_09049_b200/csrc/tc_ptx.cuh"

using namespace dg;

constexpr int PPC = 32;

__global__ void k(const __grid_constant__ CUtensorMap tm, int Cb, int n0, int h0, int w0, int r, int s, uint8_t *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bar), 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t b = ptx::smem_u32(&bar);
        ptx::mbar_arrive_expect_tx(b, (uint32_t)(PPC * Cb));
        const uint16_t ow = (uint16_t)s, oh = (uint16_t)r;
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6], {%7, %8};" ::"r"(
                ptx::smem_u32(sm)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(w0), "r"(h0), "r"(n0), "r"(b), "h"(ow), "h"(oh)
            : "memory");
        ptx::mbar_wait(b, 0);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < PPC * Cb; i += blockDim.x) out[i] = sm[i];
}

typedef CUresult (*EncIm2col)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                              const int *, const int *, cuuint32_t, cuuint32_t, const cuuint32_t *, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    void *fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fp, cudaEnableDefault, &q);
    EncIm2col enc = reinterpret_cast<EncIm2col>(fp);
    const int N = 2, H = 7, W = 9, Cb = 16, kh = 3, kw = 3, pad = 1;
    std::vector<uint8_t> X((size_t)N * H * W * Cb);
    for (size_t i = 0; i < X.size(); ++i) X[i] = (uint8_t)(i * 131 + 7) | 1;   // non-zero everywhere
    uint8_t *dx, *dout;
    cudaMalloc(&dx, X.size());
    cudaMalloc(&dout, PPC * Cb);
    cudaMemcpy(dx, X.data(), X.size(), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int stride = 1; stride <= 2; ++stride) {
        const int Ho = (H + 2 * pad - kh) / stride + 1, Wo = (W + 2 * pad - kw) / stride + 1;
        for (int up = -1; up <= -1; ++up) {   // pad - (k-1); a start outside the box traps
            CUtensorMap tm;
            cuuint64_t dims[4] = {(cuuint64_t)Cb, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
            cuuint64_t strides[3] = {(cuuint64_t)Cb, (cuuint64_t)W * Cb, (cuuint64_t)H * W * Cb};
            int lo[2] = {-pad, -pad}, hi[2] = {up, up};
            cuuint32_t es[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
            CUresult e = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, dx, dims, strides, lo, hi, Cb, PPC, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (e != CUDA_SUCCESS) {
                printf("stride %d up %d: encode failed %d\n", stride, up, (int)e);
                continue;
            }
            long bad = 0, tot = 0;
            for (int p0 = 0; p0 < N * Ho * Wo; p0 += 23) {
                const int n0 = p0 / (Ho * Wo), ho = (p0 / Wo) % Ho, wo = p0 % Wo;
                for (int r = 0; r < kh; ++r)
                    for (int s = 0; s < kw; ++s) {
                        k<<<1, 128, 64 * 1024>>>(tm, Cb, n0, ho * stride - pad, wo * stride - pad, r, s, dout);
                        std::vector<uint8_t> got(PPC * Cb);
                        cudaError_t le = cudaDeviceSynchronize();
                        if (le != cudaSuccess || cudaMemcpy(got.data(), dout, got.size(), cudaMemcpyDeviceToHost) != cudaSuccess) {
                            printf("cuda error %s (stride %d up %d p0 %d r %d s %d)\n", cudaGetErrorString(le), stride, up, p0, r, s);
                            return 1;
                        }
                        for (int i = 0; i < PPC; ++i) {
                            const int p = p0 + i;
                            if (p >= N * Ho * Wo) break;
                            const int n = p / (Ho * Wo), oh = (p / Wo) % Ho, ow = p % Wo;
                            const int hi_ = oh * stride - pad + r, wi_ = ow * stride - pad + s;
                            for (int c = 0; c < Cb; ++c) {
                                const uint8_t exp = (hi_ >= 0 && hi_ < H && wi_ >= 0 && wi_ < W)
                                                        ? X[(((size_t)n * H + hi_) * W + wi_) * Cb + c] : 0;
                                bad += got[(size_t)i * Cb + c] != exp;
                                ++tot;
                            }
                        }
                    }
            }
            printf("stride %d upper corner %d: %ld of %ld bytes wrong%s\n", stride, up, bad, tot, bad ? "" : "  <== MATCH");
        }
    }
    return 0;
}
