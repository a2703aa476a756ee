// shift_desc_test.cu — tcgen05.mma kind::i8 with both operands in shared memory in the
// no-swizzle K-major layout (16-byte rows of 16 K-codes, LBO = K-chunk stride, SBO = 128 B), the A
// descriptor started at an arbitrary ROW offset of a taller window: the "shifted view" a direct
// 3x3 conv uses to serve all taps from one unpacked input window.  Checked against the CPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/shift_desc_test tools/shift_desc_test.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../paper_2304_09049_b200/csrc/tc_ptx.cuh"

using namespace dg;

constexpr int R = 200, KK = 64, N = 64;   // window rows, K codes, N columns

__device__ __forceinline__ uint64_t desc_k_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;   // version (sm100); layout type 0 = SWIZZLE_NONE
    return d;
}

__global__ void k(const int8_t *A, const int8_t *B, int off, int32_t *D) {
    __shared__ __align__(1024) int8_t sa[R * KK];
    __shared__ __align__(1024) int8_t sb[N * KK];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // chunk j (16 codes) of row i at j * (rows * 16) + i * 16
    for (int e = threadIdx.x; e < R * KK; e += blockDim.x) {
        const int i = e / KK, kk = e % KK;
        sa[(kk / 16) * (R * 16) + i * 16 + (kk % 16)] = A[e];
    }
    for (int e = threadIdx.x; e < N * KK; e += blockDim.x) {
        const int i = e / KK, kk = e % KK;
        sb[(kk / 16) * (N * 16) + i * 16 + (kk % 16)] = B[e];
    }
    if (threadIdx.x == 0) { ptx::mbar_init(ptx::smem_u32(&bar), 1); ptx::fence_mbar_init(); }
    if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&tslot), 64);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = ptx::idesc_i8(128, N);
        const uint32_t a0 = ptx::smem_u32(sa) + off * 16, b0 = ptx::smem_u32(sb);
        for (int ks = 0; ks < KK / 32; ++ks)   // 32 codes = 2 chunks per MMA
            ptx::mma_i8_ss(tmem, desc_k_none(a0 + ks * 2 * (R * 16), R * 16, 128),
                           desc_k_none(b0 + ks * 2 * (N * 16), N * 16, 128), idesc, ks > 0);
        ptx::mma_commit(ptx::smem_u32(&bar));
    }
    ptx::mbar_wait(ptx::smem_u32(&bar), 0);
    ptx::tc_fence_after();
    uint32_t r[32];
    for (int h = 0; h < N / 32; ++h) {
        ptx::tmem_ld_32x32b_x32(tmem + h * 32 + ((uint32_t)(warp * 32) << 16), r);
        ptx::tmem_ld_wait();
        for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * N + h * 32 + j] = (int32_t)r[j];
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, 64);
}

int main() {
    int8_t hA[R * KK], hB[N * KK];
    srand(5);
    for (auto &x : hA) x = (int8_t)(rand() % 7 - 3);
    for (auto &x : hB) x = (int8_t)(rand() % 7 - 3);
    int8_t *dA, *dB;
    int32_t *dD, hD[128 * N];
    cudaMalloc(&dA, sizeof(hA));
    cudaMalloc(&dB, sizeof(hB));
    cudaMalloc(&dD, sizeof(hD));
    cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
    int fails = 0;
    for (int off : {0, 1, 7, 8, 57, 72}) {
        k<<<1, 128>>>(dA, dB, off, dD);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int i = 0; i < 128; ++i)
            for (int n = 0; n < N; ++n) {
                int s = 0;
                for (int kk = 0; kk < KK; ++kk) s += hA[(off + i) * KK + kk] * hB[n * KK + kk];
                bad += s != hD[i * N + n];
            }
        printf("row offset %3d: %s (%d mismatches)\n", off, bad ? "FAIL" : "ok", bad);
        fails += bad != 0;
    }
    return fails;
}
