// tmem_bench.cu — tcgen05.ld / tcgen05.st throughput per SM (all SMs, one CTA each).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_bench tools/tmem_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2304_09049_b200/csrc/tc_ptx.cuh"

using namespace dg;

__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr) : "memory");
}
__device__ __forceinline__ void ld32_pack16(uint32_t taddr, uint32_t (&r)[16]) {
    // 32 columns of 32-bit TMEM data read as pairs of 16-bit halves packed into 16 registers
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr) : "memory");
}

// MODE 0: x32 loads, 1: x16 loads, 2: x32.pack::16b loads, 3: x32 stores.  NW warps (multiple of 4).
template <int MODE, int NW>
__global__ void __launch_bounds__(32 * NW, 1) bench(int iters, unsigned long long *out) {
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&tslot), 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
    uint32_t acc = 0;
    __syncthreads();
    const long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const uint32_t a = base + (i & 1) * 32;
        if (MODE == 0) {
            uint32_t r[32];
            ptx::tmem_ld_32x32b_x32(a, r);
            ptx::tmem_ld_wait();
            acc += r[0] ^ r[31];
        } else if (MODE == 1) {
            uint32_t r[16];
            ld16(a, r);
            ptx::tmem_ld_wait();
            acc += r[0] ^ r[15];
        } else if (MODE == 2) {
            uint32_t r[16];
            ld32_pack16(a, r);
            ptx::tmem_ld_wait();
            acc += r[0] ^ r[15];
        } else {
            uint32_t r[32];
            for (int j = 0; j < 32; ++j) r[j] = i + j;
            ptx::tmem_st_32x32b_x32(a, r);
            ptx::tmem_st_wait();
        }
    }
    __syncthreads();
    const long long c1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = c1 - c0;
    if (acc == 0x12345) out[1] = acc;
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

template <int MODE, int NW>
void run(const char *name) {
    unsigned long long *d, h = 0;
    cudaMalloc(&d, 16);
    const int iters = 4096;
    bench<MODE, NW><<<148, 32 * NW>>>(16, d);
    bench<MODE, NW><<<148, 32 * NW>>>(iters, d);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double bytes_tmem = (MODE == 1 ? 16.0 : 32.0) * 4 * 32 * NW * iters;   // TMEM bytes touched per CTA
    printf("%-28s warps=%2d: %.1f cycles/instr/warp, %.1f TMEM bytes/cycle/SM  (%s)\n", name, NW,
           (double)h / iters, bytes_tmem / h, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    run<0, 4>("ld 32x32b.x32");
    run<0, 8>("ld 32x32b.x32");
    run<0, 16>("ld 32x32b.x32");
    run<1, 8>("ld 32x32b.x16");
    run<2, 8>("ld 32x32b.x16.pack::16b");
    run<3, 4>("st 32x32b.x32 + wait");
    run<3, 8>("st 32x32b.x32 + wait");
    run<3, 16>("st 32x32b.x32 + wait");
    return 0;
}
