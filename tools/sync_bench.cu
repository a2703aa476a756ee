// sync_bench.cu — latency of the synchronisation hops the TS kernel pipeline is built from:
//   (1) mbarrier ping-pong between two warps (arrive -> try_wait wake-up), round trip
//   (2) named barrier (bar.sync 64) ping-pong
//   (3) tcgen05.commit -> mbarrier (no MMA in flight), seen by another warp
//   (4) one 128x64x32 kind::i8 MMA + commit -> mbarrier, seen by another warp
//   (5) TMA 2-D load of a 16 KB L2-resident tile -> mbarrier
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sync_bench tools/sync_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2304_09049_b200/csrc/tc_ptx.cuh"

using namespace dg;

__global__ void __launch_bounds__(128, 1) bench(int iters, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t b1, b2, b3;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&b1), 1);
        ptx::mbar_init(ptx::smem_u32(&b2), 1);
        ptx::mbar_init(ptx::smem_u32(&b3), 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&tslot), 512);
    for (int i = threadIdx.x; i < 32768 / 16; i += 128) reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t B1 = ptx::smem_u32(&b1), B2 = ptx::smem_u32(&b2), B3 = ptx::smem_u32(&b3);
    // (1) mbarrier ping-pong
    long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (warp == 0) {
            if (lane == 0) ptx::mbar_arrive(B1);
            ptx::mbar_wait(B2, i & 1);
        } else if (warp == 1) {
            ptx::mbar_wait(B1, i & 1);
            if (lane == 0) ptx::mbar_arrive(B2);
        }
    }
    long long c1 = clock64();
    if (threadIdx.x == 0) out[0] = (c1 - c0) / iters;
    __syncthreads();
    // (2) named barrier ping-pong (warps 0, 1): two bar.sync per round
    c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (warp < 2) {
            asm volatile("bar.sync 1, 64;" ::: "memory");
            asm volatile("bar.sync 2, 64;" ::: "memory");
        }
    }
    c1 = clock64();
    if (threadIdx.x == 0) out[1] = (c1 - c0) / iters;
    __syncthreads();
    // (3) empty commit -> mbarrier seen by warp 1; warp 1 then releases warp 0 through b2
    c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (warp == 0) {
            if (lane == 0) ptx::mma_commit(B3);
            __syncwarp();
            ptx::mbar_wait(B2, i & 1);
        } else if (warp == 1) {
            ptx::mbar_wait(B3, i & 1);
            if (lane == 0) ptx::mbar_arrive(B2);
        }
    }
    c1 = clock64();
    if (threadIdx.x == 0) out[2] = (c1 - c0) / iters;
    __syncthreads();
    // (4) one MMA 128x64x32 (A from TMEM cols 256.., B zero smem) + commit
    constexpr uint32_t idesc = ptx::idesc_i8(128, 64);
    const uint64_t bdesc = ptx::desc_k_sw128(ptx::smem_u32(smem));
    c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (warp == 0) {
            if (lane == 0) {
                ptx::mma_i8_ts(tmem, tmem + 256, bdesc, idesc, 0u);
                ptx::mma_commit(B3);
            }
            __syncwarp();
            ptx::mbar_wait(B2, (iters + i) & 1);
        } else if (warp == 1) {
            ptx::mbar_wait(B3, (iters + i) & 1);
            if (lane == 0) ptx::mbar_arrive(B2);
        }
    }
    c1 = clock64();
    if (threadIdx.x == 0) out[3] = (c1 - c0) / iters;
    __syncthreads();
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

int main() {
    long long *d, h[8] = {0};
    cudaMalloc(&d, 64);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    bench<<<1, 128, 40 * 1024>>>(1000, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    printf("%s\n", cudaGetErrorString(e));
    printf("mbarrier ping-pong round trip        %lld cycles\n", h[0]);
    printf("bar.sync 64 pair (two barriers)       %lld cycles\n", h[1]);
    printf("empty commit -> mbar + mbar back     %lld cycles\n", h[2]);
    printf("1 MMA 128x64x32 + commit + mbar back %lld cycles\n", h[3]);
    return 0;
}
