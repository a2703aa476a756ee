// fp4_test.cu — go/no-go test for the e2m1 block-scaled MMA route.
//
// 2-bit activation codes a in {0..3} and weight codes w in {0..3} (levels a and w-2, BJ configs[0])
// are exact e2m1 values after halving: a/2 in {0, .5, 1, 1.5}, (w-2)/2 in {-1, -.5, 0, .5}.  With
// unit (or 2.0) ue8m0 block scales the tcgen05 kind::mxf4 MMA computes sum_k (a/2)(w-2)/2 =
// acc/4 in fp32, where acc = sum_k a*(w-2) is the exact LUT-16 GEMM value.  The question this
// program answers on the GPU is whether the tensor core's fp32 accumulation is EXACT for these
// values (|acc| <= 6*K), on random and adversarial rows, and how fast the MMA runs (SS, SW128
// K-major, M=128, N in {64,128,256}, K = 64 per instruction).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp4_test tools/fp4_test.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../paper_2304_09049_b200/csrc/tc_ptx.cuh"

using namespace dg;

// instruction descriptor, kind::mxf4 (block-scaled), e2m1 x e2m1, ue8m0 scales, K-major, dense K=64
__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
    return (1u << 7)                         // a_format = E2M1 (MXF4Format)
           | (1u << 10)                      // b_format = E2M1
           | ((uint32_t)(N >> 3) << 17)      // N / 8
           | (1u << 23)                      // scale format UE8M0
           | ((uint32_t)(M >> 4) << 24);     // M / 16
}

DG_DEV void mma_mxf4(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc, uint32_t sfa, uint32_t sfb) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb)
        : "memory");
}

// A image: [K/256 atoms][128 rows][128 B] SW128; B image: [K/256][N][128 B].  One CTA, 128 threads.
template <int N>
__global__ void __launch_bounds__(128, 1) fp4_gemm(const uint8_t *aimg, const uint8_t *bimg, int K, uint32_t sfbyte,
                                                   float *D, int reps, unsigned long long *cyc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int natoms = (K + 255) / 256;
    const int abytes = natoms * 128 * 128, bbytes = natoms * N * 128;
    for (int i = threadIdx.x; i < abytes / 16; i += 128) reinterpret_cast<uint4 *>(smem)[i] = reinterpret_cast<const uint4 *>(aimg)[i];
    for (int i = threadIdx.x; i < bbytes / 16; i += 128)
        reinterpret_cast<uint4 *>(smem + abytes)[i] = reinterpret_cast<const uint4 *>(bimg)[i];
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bar), 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&tslot), 512);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    // scale factors: columns [256, 288) of every lane = sfbyte replicated (any SF layout reads it)
    {
        uint32_t r[32];
        for (int j = 0; j < 32; ++j) r[j] = sfbyte * 0x01010101u;
        ptx::tmem_st_32x32b_x32(tmem + 256 + ((uint32_t)(warp * 32) << 16), r);
        ptx::tmem_st_wait();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t sfa = tmem + 256, sfb = tmem + 272;
    if (threadIdx.x == 0) {
        const uint64_t ad0 = ptx::desc_k_sw128(ptx::smem_u32(smem)), bd0 = ptx::desc_k_sw128(ptx::smem_u32(smem + abytes));
        const int nk = K / 64;
        const unsigned long long t0 = clock64();
        for (int rep = 0; rep < reps; ++rep)
            for (int k = 0; k < nk; ++k)
                mma_mxf4(tmem, ad0 + (uint64_t)(((k >> 2) * 128 * 128) >> 4) + 2 * (k & 3),
                         bd0 + (uint64_t)(((k >> 2) * N * 128) >> 4) + 2 * (k & 3), idesc_mxf4(128, N), (k > 0 || rep > 0) ? 1u : 0u,
                         sfa, sfb);
        ptx::mma_commit(ptx::smem_u32(&bar));
        ptx::mbar_wait(ptx::smem_u32(&bar), 0);
        cyc[0] = clock64() - t0;
    }
    __syncthreads();
    ptx::tc_fence_after();
    for (int c = 0; c < N; c += 32) {
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tmem + c + ((uint32_t)(warp * 32) << 16), r);
        ptx::tmem_ld_wait();
        for (int j = 0; j < 32; ++j) D[(size_t)threadIdx.x * N + c + j] = __uint_as_float(r[j]);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

static uint64_t s_rng = 0x9E3779B97F4A7C15ull;
static uint32_t rnd() {
    s_rng ^= s_rng << 13; s_rng ^= s_rng >> 7; s_rng ^= s_rng << 17;
    return (uint32_t)(s_rng >> 11);
}

// e2m1 nibble of value v/2 for the integer level v in [-2, 3]
static uint8_t nib_half(int v) {
    static const uint8_t pos[4] = {0x0, 0x1, 0x2, 0x3};   // 0, .5, 1, 1.5
    return v >= 0 ? pos[v] : (uint8_t)(0x8 | pos[-v]);
}

// SW128 K-major image of R rows x K fp4 values (element k of row r: nibble k&1 of byte k>>1 in the
// row's K-atom k>>8, 16-byte chunk ((k&255)>>5) ^ (r&7))
static void make_image(const std::vector<int> &v, int R, int K, std::vector<uint8_t> &img) {
    img.assign((size_t)((K + 255) / 256) * R * 128, 0);
    for (int r = 0; r < R; ++r)
        for (int k = 0; k < K; ++k) {
            const int atom = k >> 8, kk = k & 255, byte = kk >> 1, chunk = byte >> 4;
            const size_t off = (size_t)atom * R * 128 + (size_t)r * 128 + (size_t)(((chunk ^ (r & 7)) << 4) | (byte & 15));
            img[off] |= (uint8_t)(nib_half(v[(size_t)r * K + k]) << (4 * (k & 1)));
        }
}

template <int N>
static int run(int K, int pattern, uint32_t sfbyte, int reps) {
    std::vector<int> A((size_t)128 * K), B((size_t)N * K);   // A: activation levels 0..3; B: weight levels -2..1
    for (int r = 0; r < 128; ++r)
        for (int k = 0; k < K; ++k) {
            int a = rnd() & 3;
            if (pattern == 1 && (r & 1) && k < K - 64) a = 3;                       // big partial sums first
            if (pattern == 2 && (r & 3) == 1) a = (k & 1) ? 3 : 0;
            A[(size_t)r * K + k] = a;
        }
    for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) {
            int w = (int)(rnd() & 3) - 2;
            if (pattern == 1 && (n & 1) && k < K - 64) w = -2;
            if (pattern == 2 && (n & 3) == 1) w = (k & 2) ? 1 : -2;
            B[(size_t)n * K + k] = w;
        }
    std::vector<uint8_t> ai, bi;
    make_image(A, 128, K, ai);
    make_image(B, N, K, bi);
    uint8_t *da, *db;
    float *dd;
    unsigned long long *dc;
    cudaMalloc(&da, ai.size());
    cudaMalloc(&db, bi.size());
    cudaMalloc(&dd, (size_t)128 * N * 4);
    cudaMalloc(&dc, 64);
    cudaMemcpy(da, ai.data(), ai.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(db, bi.data(), bi.size(), cudaMemcpyHostToDevice);
    const int smem = (int)(ai.size() + bi.size()) + 1024;
    cudaFuncSetAttribute(fp4_gemm<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    fp4_gemm<N><<<1, 128, smem>>>(da, db, K, sfbyte, dd, reps, dc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("N=%d K=%d: CUDA error %s\n", N, K, cudaGetErrorString(e));
        return 1;
    }
    std::vector<float> D((size_t)128 * N);
    unsigned long long cyc;
    cudaMemcpy(D.data(), dd, D.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    // expected: reps * sum_k A*B * s^2 / 4, s = 2^(sfbyte - 127)
    const double s = ldexp(1.0, (int)sfbyte - 127);
    long bad = 0, maxabs = 0;
    double first_got = 0, first_exp = 0;
    for (int r = 0; r < 128; ++r)
        for (int n = 0; n < N; ++n) {
            long acc = 0;
            for (int k = 0; k < K; ++k) acc += (long)A[(size_t)r * K + k] * B[(size_t)n * K + k];
            maxabs = labs(acc) > maxabs ? labs(acc) : maxabs;
            const double exp = (double)reps * acc * s * s / 4.0;
            const double got = D[(size_t)r * N + n];
            if (got != exp) {
                if (!bad) { first_got = got; first_exp = exp; }
                ++bad;
            }
        }
    printf("N=%3d K=%5d pattern=%d sf=%u reps=%d: %s (%ld of %d wrong; max|acc| %ld)%s cycles/MMA %.1f\n", N, K, pattern,
           sfbyte, reps, bad ? "MISMATCH" : "exact", bad, 128 * N, maxabs, "", (double)cyc / ((double)reps * K / 64));
    if (bad) printf("   first mismatch got %.6f expected %.6f\n", first_got, first_exp);
    cudaFree(da); cudaFree(db); cudaFree(dd); cudaFree(dc);
    return bad ? 1 : 0;
}

int main() {
    int fails = 0;
    for (int pattern = 0; pattern < 3; ++pattern) {
        fails += run<64>(576, pattern, 127, 1);
        fails += run<64>(4608 / 2, pattern, 127, 1);
        fails += run<128>(1152, pattern, 128, 1);
        fails += run<128>(1024, pattern, 127, 1);
        fails += run<256>(512, pattern, 127, 1);
    }
    // long accumulations (|acc| up to reps * 6K) and throughput
    fails += run<64>(512, 1, 127, 9);
    fails += run<128>(512, 1, 128, 9);
    fails += run<256>(512, 1, 127, 9);
    fails += run<64>(256, 0, 127, 200);
    fails += run<128>(256, 0, 127, 200);
    fails += run<256>(256, 0, 127, 200);
    printf("%s\n", fails ? "FP4 ROUTE: NOT EXACT" : "FP4 ROUTE: all exact");
    return 0;
}
