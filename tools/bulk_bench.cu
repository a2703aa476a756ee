// bulk_bench.cu — HBM read rate of cp.async.bulk (1-D bulk copies) into a ring of shared-memory
// slots, one issuing thread per CTA (148 CTAs), as a function of copy size and ring depth.
// A slot is reused only after its mbarrier completed (the consumer is the issuing warp itself).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bulk_bench tools/bulk_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2304_09049_b200/csrc/tc_ptx.cuh"

using namespace dg;

__global__ void __launch_bounds__(32, 1) bench(const uint8_t *src, size_t per_cta, int bytes, int slots, int whole_warp) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[64];
    const int lane = threadIdx.x;
    if (lane == 0) {
        for (int i = 0; i < slots; ++i) ptx::mbar_init(ptx::smem_u32(&bars[i]), 1);
        ptx::fence_mbar_init();
    }
    __syncwarp();
    const uint8_t *base = src + (size_t)blockIdx.x * per_cta;
    const int n = (int)(per_cta / bytes);
    for (int i = 0; i < n; ++i) {
        const int slot = i % slots;
        if (i >= slots) ptx::mbar_wait(ptx::smem_u32(&bars[slot]), (uint32_t)((i / slots - 1) & 1));   // copy i - slots done
        if (lane == 0) {
            ptx::mbar_arrive_expect_tx(ptx::smem_u32(&bars[slot]), (uint32_t)bytes);
            ptx::bulk_load(ptx::smem_u32(smem + (size_t)slot * bytes), base + (size_t)i * bytes, (uint32_t)bytes,
                           ptx::smem_u32(&bars[slot]));
        }
        __syncwarp();
    }
    for (int i = (n > slots ? n - slots : 0); i < n; ++i)   // drain before the smem goes away
        ptx::mbar_wait(ptx::smem_u32(&bars[i % slots]), (uint32_t)((i / slots) & 1));
    if (!whole_warp) return;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t total = (size_t)2 << 30;
    uint8_t *d = nullptr;
    if (cudaMalloc(&d, total) != cudaSuccess) { printf("malloc failed\n"); return 1; }
    cudaMemset(d, 1, total);
    printf("sms %d\n", sms);
    fflush(stdout);
    const size_t per_cta = total / sms / 65536 * 65536;
    cudaError_t ea = cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    printf("attr %s\n", cudaGetErrorString(ea));
    fflush(stdout);
    const int sizes[] = {2048, 4096, 8192, 16384};
    const int depths[] = {4, 8, 16, 32};
    for (int s : sizes)
        for (int dep : depths) {
            if ((size_t)s * dep > 128 * 1024) continue;
            bench<<<sms, 32, s * dep>>>(d, per_cta, s, dep, 1);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            bench<<<sms, 32, s * dep>>>(d, per_cta, s, dep, 1);
            cudaEventRecord(e1);
            cudaError_t es = cudaEventSynchronize(e1);
            if (es != cudaSuccess) { printf("kernel error %s\n", cudaGetErrorString(es)); return 1; }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("copy %6d B x %2d slots in flight: %7.1f GB/s  (%s)\n", s, dep, per_cta * sms / (ms * 1e-3) / 1e9,
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
