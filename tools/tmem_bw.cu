// tmem_bw.cu — TMEM read bandwidth per SM as the epilogue of a 128 x 256 accumulator sees it
// (all SMs, one CTA each; NW warps, warp w reads lane quarter w % 4, column group w / 4).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I. -o tools/tmem_bw tools/tmem_bw.cu
// Modes: 0 x32 per wait (32 columns), 1 two x32 per wait (64 columns in flight),
//        2 x32.pack::16b per wait (64 columns -> 32 registers), 3 two x32.pack::16b per wait,
//        4 16x256b.x8 per wait (cells: 16 lanes x 8 x 256 bits = 32 columns of 16 lanes x2)
// Reported: 32-bit TMEM cells read per cycle per SM x 4 bytes.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2304_09049_b200/csrc/tc_ptx.cuh"

using namespace dg;

template <int MODE, int NW>
__global__ void __launch_bounds__(32 * NW, 1) bench(int iters, unsigned long long *out) {
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&tslot), 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128) % 512;
    uint32_t acc = 0;
    __syncthreads();
    const long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const uint32_t a = base + (uint32_t)((i & 1) * 64);
        uint32_t r[32], s[32];
        if (MODE == 0) {
            ptx::tmem_ld_32x32b_x32(a, r);
            ptx::tmem_ld_wait();
            acc += r[0] ^ r[31];
        } else if (MODE == 1) {
            ptx::tmem_ld_32x32b_x32(a, r);
            ptx::tmem_ld_32x32b_x32(a + 32, s);
            ptx::tmem_ld_wait();
            acc += r[0] ^ r[31] ^ s[0] ^ s[31];
        } else if (MODE == 2) {
            ptx::tmem_ld_32x32b_x32_pack16(a, r);
            ptx::tmem_ld_wait();
            acc += r[0] ^ r[31];
        } else if (MODE == 3) {
            ptx::tmem_ld_32x32b_x32_pack16(a, r);
            ptx::tmem_ld_32x32b_x32_pack16(a + 64, s);
            ptx::tmem_ld_wait();
            acc += r[0] ^ r[31] ^ s[0] ^ s[31];
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
    const double cols = MODE == 0 ? 32 : (MODE == 3 ? 128 : 64);
    const double cells = cols * 32 * NW * iters;   // 32-bit TMEM cells read per CTA
    printf("%-34s warps=%2d: %7.1f cycles/iter/warp, %6.1f TMEM B/cycle/SM  (%s)\n", name, NW, (double)h / iters,
           4 * cells / h, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    run<0, 4>("x32 (32 col) + wait");
    run<0, 8>("x32 (32 col) + wait");
    run<0, 16>("x32 (32 col) + wait");
    run<1, 4>("2 x32 (64 col) + wait");
    run<1, 8>("2 x32 (64 col) + wait");
    run<2, 4>("x32.pack16 (64 col) + wait");
    run<2, 8>("x32.pack16 (64 col) + wait");
    run<2, 16>("x32.pack16 (64 col) + wait");
    run<3, 4>("2 x32.pack16 (128 col) + wait");
    run<3, 8>("2 x32.pack16 (128 col) + wait");
    return 0;
}
