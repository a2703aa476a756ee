// tmem_pack_test.cu — semantics of tcgen05.ld.32x32b.x16.pack::16b (which columns land in
// which 16-bit half) and of VIADDMNMX.S16x2.RELU overflow behaviour.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_pack_test tools/tmem_pack_test.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2304_09049_b200/csrc/tc_ptx.cuh"

using namespace dg;

__global__ void k(uint32_t *out, uint32_t *out2) {
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&tslot), 32);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) v[c] = (uint32_t)(lane * 1000 + c - 500) ;
    ptx::tmem_st_32x32b_x32(tmem, v);
    ptx::tmem_st_wait();
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(tmem) : "memory");
    ptx::tmem_ld_wait();
    for (int i = 0; i < 16; ++i) out[lane * 16 + i] = r[i];
    // VIADDMNMX.RELU: x = max(min(a + b, c), 0) per 16-bit lane, probe overflow
    const uint32_t a = 0x7F00u | (0x8100u << 16), b = 0x0200u | (0xFE00u << 16);
    out2[lane] = __viaddmin_s16x2_relu(a + lane, b, 0x7FFF7FFFu);
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, 32);
}

int main() {
    uint32_t *d, *d2, h[512], h2[32];
    cudaMalloc(&d, 2048);
    cudaMalloc(&d2, 128);
    k<<<1, 32>>>(d, d2);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, 2048, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2, d2, 128, cudaMemcpyDeviceToHost);
    for (int l = 0; l < 2; ++l) {
        printf("lane %d:", l);
        for (int i = 0; i < 16; ++i) printf(" [%d|%d]", (int)(int16_t)(h[l * 16 + i] & 0xFFFF), (int)(int16_t)(h[l * 16 + i] >> 16));
        printf("\n");
    }
    printf("viaddmin_relu(0x7F00+lane, 0x0200) lo/hi lane0: %d %d\n", (int)(int16_t)(h2[0] & 0xFFFF), (int)(int16_t)(h2[0] >> 16));
    return 0;
}
