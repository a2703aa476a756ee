// mma_bench.cu — tcgen05.mma kind::i8 throughput microbenchmark (one CTA per SM, all SMs).
// Issues NITER back-to-back MMAs (M=128, N in {64,128,256}, K=32) from one thread with A from
// TMEM (TS) or shared memory (SS), commits once, waits, and reports cycles per MMA and the
// chip-wide int8 TOPS.  Operand contents are zero (throughput does not depend on values).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../paper_2304_09049_b200/csrc/tc_ptx.cuh"

using namespace dg;

__device__ __forceinline__ bool lane_is_zero() { return (threadIdx.x & 31) == 0; }

// MODE 0: MMA only; 1: + 4 warps of tcgen05.st (32 cols) loops; 2: + 4 warps of LDS.128 loops;
// 3: + 4 warps of tcgen05.ld (32 cols) loops; 4: commit every 4 MMAs; 5: 4 + try_wait on a
// completed barrier + fence::after_thread_sync every 4 MMAs; 6: two commits every 4 MMAs
template <int N, bool TS, int MODE>
__global__ void __launch_bounds__(256, 1) bench(int niter, unsigned long long *cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar, bar2[4], bar_done;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (128 + N) * 128 / 16; i += blockDim.x) {
        // MODE 24/25/26: random operand bytes (int8 levels in [-2, 3] / full range) instead of zeros
        uint32_t h[4];
        for (int j = 0; j < 4; ++j) {
            uint32_t x = (uint32_t)(i * 4 + j) * 0x9E3779B1u + 0x7F4A7C15u;
            x ^= x >> 15; x *= 0x2C1B3C6Du; x ^= x >> 12; x *= 0x297A2D39u; x ^= x >> 15;
            h[j] = MODE == 26 ? x : ((x & 0x03030303u) - (i < 128 * 8 ? 0u : 0x02020202u));
        }
        reinterpret_cast<uint4 *>(smem)[i] = (MODE >= 24 && MODE <= 26) ? make_uint4(h[0], h[1], h[2], h[3]) : make_uint4(0, 0, 0, 0);
    }
    if (threadIdx.x == 0) {
        ptx::mbar_init(ptx::smem_u32(&bar), 1);
        ptx::mbar_init(ptx::smem_u32(&bar_done), 1);
        for (int j = 0; j < 4; ++j) ptx::mbar_init(ptx::smem_u32(&bar2[j]), 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) ptx::tmem_alloc(ptx::smem_u32(&tslot), 512);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    if (TS && MODE >= 24 && MODE <= 26 && warp < 4) {   // random A operand in TMEM columns [256, 288)
        uint32_t r[32];
        for (int j = 0; j < 32; ++j) {
            uint32_t x = (uint32_t)(threadIdx.x * 32 + j) * 0x9E3779B1u + 0x1234567u;
            x ^= x >> 15; x *= 0x2C1B3C6Du; x ^= x >> 12; x *= 0x297A2D39u; x ^= x >> 15;
            r[j] = MODE == 26 ? x : (x & 0x03030303u);
        }
        ptx::tmem_st_32x32b_x32(tmem + 256 + ((uint32_t)(warp * 32) << 16), r);
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
    }
    __syncthreads();
    ptx::tc_fence_after();
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    __syncthreads();
    if (threadIdx.x == 0) ptx::mbar_arrive(ptx::smem_u32(&bar_done));   // phase 0 complete
    __syncthreads();
    // MODE 27: 7 ALU-bound warps (1..7) beside the MMA thread of warp 0 (the lowest scheduling
    // priority); MODE 28: the MMA thread in warp 7 (the highest id), ALU warps 0..6
    constexpr int MMA_TID = MODE == 28 ? 224 : 0;
    // MODE 29: ALU warps only on the OTHER sub-partitions (warps 1..3, 5..7: the MMA warp 0 shares
    // SMSP 0 with nobody busy); MODE 30: a single ALU warp (4) on the MMA warp's sub-partition
    if ((MODE == 27 && warp >= 1) || (MODE == 28 && warp < 7) || (MODE == 29 && (warp & 3) != 0) || ((MODE == 30 || MODE == 31) && warp == 4)) {
        uint32_t x[8];
        for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
        while (!done) {
#pragma unroll
            for (int r = 0; r < 16; ++r)
#pragma unroll
                for (int j = 0; j < 8; ++j) x[j] = x[j] * 0x9E3779B1u + (x[j] >> 7);
        }
        if ((x[0] ^ x[1] ^ x[2] ^ x[3] ^ x[4] ^ x[5] ^ x[6] ^ x[7]) == 12345u) cycles[3] = 1;
    }
    if (warp >= 4 && (MODE == 22 || MODE == 23)) {   // smem store / load traffic from other warps
        uint32_t *buf = reinterpret_cast<uint32_t *>(smem + (128 + N) * 128);   // 16 KB after the operands
        unsigned acc = 0;
        int it = 0;
        while (!done) {
            const int o = ((it * 64 + (threadIdx.x - 128) * 4) & 4095);
            if (MODE == 22) *reinterpret_cast<uint4 *>(buf + o) = make_uint4(it, it, it, it);
            else { const uint4 v = *reinterpret_cast<const uint4 *>(buf + o); acc += v.x; }
            ++it;
        }
        if (acc == 12345) cycles[3] = acc;
    }
    if (warp >= 4 && MODE >= 1 && MODE <= 3) {   // interference warps, lane quarter = warp % 4
        const uint32_t taddr = tmem + 448 + ((uint32_t)((warp & 3) * 32) << 16);
        uint32_t r[32];
        for (int j = 0; j < 32; ++j) r[j] = j;
        unsigned acc = 0;
        int it = 0;
        while (!done) {
            if (MODE == 1) {
                ptx::tmem_st_32x32b_x32(taddr, r);
                ptx::tmem_st_wait();
            } else if (MODE == 2) {
                const uint4 v = reinterpret_cast<const uint4 *>(smem)[((it * 37 + threadIdx.x) & 1023)];
                acc += v.x ^ v.y;
            } else {
                ptx::tmem_ld_32x32b_x32(taddr, r);
                ptx::tmem_ld_wait();
                acc += r[3];
                if (MODE == 16) {
                    uint4 *gp = reinterpret_cast<uint4 *>(cycles + 64) + ((blockIdx.x * 256 + threadIdx.x) & 4095);
                    *gp = make_uint4(r[0], r[1], r[2], r[4]);
                }
            }
            ++it;
        }
        if (acc == 12345) cycles[3] = acc;
    }
    if (MODE == 13 && warp == 1) {
        for (int i = 0; i < niter; i += 4) {
            ptx::mbar_wait(ptx::smem_u32(&bar_done), 0);
            asm volatile("bar.sync 2, 64;" ::: "memory");
        }
    }
    if (MODE >= 11 && MODE <= 13 && warp == 0) {
        const uint32_t a = ptx::smem_u32(smem), b = a + 128 * 128;
        constexpr uint32_t idesc = ptx::idesc_i8(128, N);
        const long long c0 = clock64();
        for (int i = 0; i < niter; ++i) {
            const int k = i & 3;
            if (k == 0) {
                if (MODE == 11) ptx::mbar_wait(ptx::smem_u32(&bar_done), 0);
                if (MODE == 12) asm volatile("bar.sync 1, 32;" ::: "memory");
                if (MODE == 13) asm volatile("bar.sync 2, 64;" ::: "memory");
                ptx::tc_fence_after();
            }
            if (threadIdx.x == 0) ptx::mma_i8_ts(tmem, tmem + 256 + 8 * k, ptx::desc_k_sw128(b + 32 * k), idesc, i > 0);
            __syncwarp();
        }
        const long long c1 = clock64();
        if (threadIdx.x == 0) {
            ptx::mma_commit(ptx::smem_u32(&bar));
            ptx::mbar_wait(ptx::smem_u32(&bar), 0);
        }
        __syncwarp();
        const long long c2 = clock64();
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            cycles[0] = c1 - c0;
            cycles[1] = c2 - c0;
        }
        if (threadIdx.x == 0) done = 1;
    }
    // MODE 31 (one ALU warp on SMSP 0) / 32 (none): the whole of warp 0 issues 4 MMAs per asm block,
    // elect.sync inside and the per-MMA operand offsets added in PTX (uniform datapath), instead of
    // one asm statement per MMA under `if (lane == 0)` (3 R2UR + ELECT loop per MMA)
    if ((MODE == 31 || MODE == 32) && warp == 0) {
        const uint32_t b = ptx::smem_u32(smem) + 128 * 128;
        constexpr uint32_t idesc = ptx::idesc_i8(128, N);
        const uint64_t bd = ptx::desc_k_sw128(b);
        const uint32_t at = tmem + 256;
        const long long c0 = clock64();
        for (int i = 0; i < niter; i += 4) {
            asm volatile(
                "{\n\t.reg .pred p;\n\t.reg .b32 a1, a2, a3;\n\t.reg .b64 b1, b2, b3;\n\t"
                "elect.sync _|p, 0xffffffff;\n\t"
                "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
                "add.u64 b1, %2, 2;\n\tadd.u64 b2, %2, 4;\n\tadd.u64 b3, %2, 6;\n\t"
                "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;\n\t"
                "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %3, 1;\n\t"
                "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [a2], b2, %3, 1;\n\t"
                "@p tcgen05.mma.cta_group::1.kind::i8 [%0], [a3], b3, %3, 1;\n\t}"
                ::"r"(tmem), "r"(at), "l"(bd), "r"(idesc)
                : "memory");
        }
        const long long c1 = clock64();
        if (lane_is_zero()) {
            ptx::mma_commit(ptx::smem_u32(&bar));
            ptx::mbar_wait(ptx::smem_u32(&bar), 0);
        }
        __syncwarp();
        const long long c2 = clock64();
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            cycles[0] = c1 - c0;
            cycles[1] = c2 - c0;
        }
        if (threadIdx.x == 0) done = 1;
    }
    if (threadIdx.x == MMA_TID && (MODE < 11 || MODE >= 14) && MODE != 31 && MODE != 32) {
        const uint32_t a = ptx::smem_u32(smem), b = a + 128 * 128;
        constexpr uint32_t idesc = ptx::idesc_i8(128, N);
        const long long c0 = clock64();
        for (int i = 0; i < niter; ++i) {
            const int k = i & 3;
            if (MODE == 5 && k == 0) {
                ptx::mbar_wait(ptx::smem_u32(&bar_done), 0);
                ptx::tc_fence_after();
            }
            if (MODE == 7 && k == 0) ptx::mbar_wait(ptx::smem_u32(&bar_done), 0);
            if (MODE == 8 && k == 0) ptx::tc_fence_after();
            if (MODE == 9 && k == 0) {   // test_wait (non-blocking probe) instead of try_wait
                uint32_t ok;
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok) : "r"(ptx::smem_u32(&bar_done)), "r"(0u) : "memory");
                if (!ok) ptx::mbar_wait(ptx::smem_u32(&bar_done), 0);
            }
            if (MODE == 10 && k == 0) {   // volatile smem flag poll instead of an mbarrier
                while (done == 7) {}
            }
            if (TS)
                ptx::mma_i8_ts(tmem, tmem + 256 + 8 * k, ptx::desc_k_sw128(b + 32 * k), idesc, i > 0);
            else if (MODE == 20)   // A in the no-swizzle K-major layout (16-byte rows, LBO = 128 rows * 16 B)
                ptx::mma_i8_ss(tmem, ptx::desc_k_none(a + (uint32_t)(k & 1) * 2 * 2048, 2048), ptx::desc_k_sw128(b + 32 * k), idesc, i > 0);
            else if (MODE == 21 || MODE == 22 || MODE == 23 || MODE == 25)   // A no-swizzle, shifted by 57 rows (window view)
                ptx::mma_i8_ss(tmem, ptx::desc_k_none(a + 57 * 16 + (uint32_t)(k & 1) * 2 * 2048, 2048), ptx::desc_k_sw128(b + 32 * k), idesc, i > 0);
            else
                ptx::mma_i8_ss(tmem, ptx::desc_k_sw128(a + 32 * k), ptx::desc_k_sw128(b + 32 * k), idesc, i > 0);
            if ((MODE == 4 || MODE == 5 || MODE == 6) && k == 3) ptx::mma_commit(ptx::smem_u32(&bar2[(i >> 2) & 3]));
            if (MODE == 6 && k == 3) ptx::mma_commit(ptx::smem_u32(&bar2[((i >> 2) + 1) & 3]));
        }
        const long long c1 = clock64();
        ptx::mma_commit(ptx::smem_u32(&bar));
        ptx::mbar_wait(ptx::smem_u32(&bar), 0);
        const long long c2 = clock64();
        if (blockIdx.x == 0) {   // (MODE 27/28 write from their own MMA thread)
            cycles[0] = c1 - c0;
            cycles[1] = c2 - c0;
        }
        done = 1;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, 512);
}

template <int N, bool TS, int MODE = 0>
void run(int sms) {
    const int niter = 20000;
    unsigned long long *d;
    cudaMalloc(&d, 16 + 64 * 8 + 4096 * 16 + 1024);
    const int smem = (128 + N) * 128 + 16384;
    cudaFuncSetAttribute(bench<N, TS, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    bench<N, TS, MODE><<<sms, 256, smem>>>(100, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench<N, TS, MODE><<<sms, 256, smem>>>(niter, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double ops = 2.0 * 128 * N * 32 * (double)niter * sms;
    printf("N %d mode=%d kind::i8 M=128 %s: issue %.1f cyc/mma, complete %.1f cyc/mma, %.1f TOPS chip (%d CTAs, %.3f ms) %s\n", N,
           MODE, TS ? "A=TMEM" : "A=SMEM", (double)h[0] / niter, (double)h[1] / niter, ops / (ms * 1e-3) / 1e12, sms, ms,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main(int argc, char **argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<64, true>(sms);
    run<128, true>(sms);
    run<256, true>(sms);
    run<128, false>(sms);
    run<256, false>(sms);
    run<64, false, 20>(sms);
    run<128, false, 20>(sms);
    run<64, false, 21>(sms);
    run<64, false>(sms);
    run<64, false, 22>(sms);
    run<64, false, 23>(sms);
    // data dependence: random operands (24: levels, 25: levels + shifted no-swizzle A, 26: random bytes)
    run<64, true, 24>(sms);
    run<128, true, 24>(sms);
    run<256, true, 24>(sms);
    run<64, false, 24>(sms);
    run<128, false, 24>(sms);
    run<256, false, 24>(sms);
    run<64, false, 25>(sms);
    run<64, true, 26>(sms);
    run<128, true, 26>(sms);
    run<256, true, 26>(sms);
    run<128, false, 26>(sms);
    // issue pressure: ALU-bound warps beside the MMA-issuing thread
    run<64, true, 27>(sms);
    run<64, true, 28>(sms);
    run<128, true, 27>(sms);
    run<128, true, 28>(sms);
    run<64, true, 29>(sms);
    run<64, true, 30>(sms);
    run<128, true, 29>(sms);
    run<128, true, 30>(sms);
    run<64, true, 2>(sms);
    run<64, true, 31>(sms);
    run<64, true, 32>(sms);
    run<128, true, 31>(sms);
    run<128, true, 32>(sms);
    if (argc > 1) {   // pipeline-interaction modes (see MODE above)
        run<64, true, 1>(sms);
        run<64, true, 3>(sms);
        run<64, true, 4>(sms);
        run<64, true, 5>(sms);
        run<64, true, 6>(sms);
        run<64, true, 8>(sms);
        run<64, true, 13>(sms);
        run<128, true, 1>(sms);
        run<128, true, 4>(sms);
        run<128, true, 5>(sms);
    }
    return 0;
}
