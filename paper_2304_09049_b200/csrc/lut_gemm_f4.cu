// lut_gemm_f4.cu — the LUT-16 GEMM for 2-bit product tables on the block-scaled FP4 tensor-core
// path (tcgen05 kind::mxf4, e2m1 x e2m1):
//
//   C[m][n] = sum_{k<K} T[(W[m][k] << 2) | A[k][n]] = sum_k wl[W[m][k]] * al[A[k][n]]
//
// For activation levels al = {0, 1, 2, 3} (BJ configs 1-4) the activation CODE c is already the
// e2m1 encoding of the value c/2 (e2m1 0000 = 0, 0001 = 0.5, 0010 = 1, 0011 = 1.5), so the
// paper's unpack step (Alg. 1 line 9: mask / shift the packed codes) becomes two nibble
// masks per 16 codes: x & 0x33333333 (the even codes) and (x >> 2) & 0x33333333 (the odd ones).
// Weight levels v with v/2 in e2m1 ({0, +-1, +-2, +-3, +-4, +-6, +-8, +-12}) are expanded once
// (offline, like the paper's weight packing) to e2m1 nibbles of v/2 in the same order.
// Unit-power block scales 2 x 2 make the tensor core's fp32 sum equal sum(a*w) exactly: every
// partial sum is an integer below 2^22, and tools/fp4_test.cu checks that the hardware
// accumulation is exact on random and adversarial rows (profiles/r01_fp4_mxf4_test.txt).
//
// Tile: 128 activation rows (n) x 240 weight rows (m); D[n][m] in TMEM (fp32, two buffers), stored
// transposed into C[m][n] (each store instruction writes 32 consecutive n of one m: coalesced).
// Persistent, warp-specialised, one CTA per SM:
//   warps 0..3  epilogue (lane quarter = warp): TMEM -> exact int32 -> C
//   warps 4..7  unpack: thread = activation row; packed smem slot -> e2m1 nibbles -> SW128 A stage
//   warp 8      producer: TMA of packed A slots (512 codes per row) and e2m1 B stages (256 codes)
//   warp 9      waiter: mbarrier waits, hands each stage to the MMA warp through a named barrier
//   warp 10     MMA issuer (whole warp, one lane elected inside the asm)
#include <cuda.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace dg {
namespace {

constexpr int F4_BM = 128;           // activation rows per tile (MMA M, TMEM lanes)
constexpr int F4_BN = 240;           // weight rows per tile (MMA N): 2 x 240 fp32 accumulator columns + 32
                                     // block-scale columns fill the 512 TMEM columns
constexpr int F4_KST = 256;          // codes per pipeline stage = 128 bytes of e2m1 per row = 4 MMAs
constexpr int F4_SA = 4, F4_SB = 4, F4_SP = 2, F4_NACC = 2;
constexpr int F4_A_STAGE = F4_BM * F4_KST / 2;     // 16 KB, SW128 K-major
constexpr int F4_B_STAGE = F4_BN * F4_KST / 2;     // 32 KB, SW128 K-major
constexpr int F4_P_SLOT = F4_BM * 128;             // 16 KB: 512 packed codes per row (2 stages)
constexpr int F4_OFF_B = 0;
constexpr int F4_OFF_A = F4_OFF_B + F4_SB * F4_B_STAGE;
constexpr int F4_OFF_P = F4_OFF_A + F4_SA * F4_A_STAGE;
constexpr int F4_OFF_BAR = F4_OFF_P + F4_SP * F4_P_SLOT;
constexpr int F4_NBAR = 2 * F4_SP + 2 * F4_SB + 2 * F4_SA + 2 * F4_NACC;
constexpr int F4_OFF_TMEM = F4_OFF_BAR + F4_NBAR * 8;
constexpr int F4_ALLOC = F4_OFF_TMEM + 16 + 1024;
static_assert(F4_ALLOC <= 232448, "shared memory budget");
constexpr int F4_EPI0 = 0, F4_UNP0 = 4, F4_PROD = 8, F4_WAIT = 9, F4_MMA = 10, F4_NT = 32 * 11;
constexpr int F4_HANDOFF_BAR = 1;
constexpr uint32_t F4_SF_COL = 480;  // TMEM columns [480, 512): block scales (every byte 2^1)

// instruction descriptor: kind::mxf4, e2m1 x e2m1, ue8m0 scales, K-major, dense K = 64
__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
    return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}

DG_DEV void mma_mxf4_warp(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc, uint32_t sfa, uint32_t sfb) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb)
        : "memory");
}

struct F4Args {
    int64_t M, N, ldc;
    int32_t nstages, last_ksteps, ntn, ntm, ntiles;
    int32_t *C;
};

// tile t -> (activation block tn, weight block tm), walked in groups of F4_GROUP activation blocks
// x all weight blocks (weight block outer inside a group): a wave of concurrent tiles touches ~16
// activation blocks and ~10 weight blocks, so both operands stay L2-resident across the wave
constexpr int F4_GROUP = 16;
DG_DEV void f4_tile(const F4Args &fa, int t, int &tn, int &tm) {
    const int grp = t / (F4_GROUP * fa.ntm), rem = t - grp * (F4_GROUP * fa.ntm);
    const int gl = fa.ntn - grp * F4_GROUP < F4_GROUP ? fa.ntn - grp * F4_GROUP : F4_GROUP;
    tm = rem / gl;
    tn = grp * F4_GROUP + (rem - tm * gl);
}

__global__ void __launch_bounds__(F4_NT, 1)
lut_gemm_f4_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                   const __grid_constant__ F4Args fa) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = ptx::smem_u32(smem);
    const uint32_t bar0 = sbase + F4_OFF_BAR;
    auto full_p = [&](int s) { return bar0 + 8 * s; };
    auto empty_p = [&](int s) { return bar0 + 8 * (F4_SP + s); };
    auto full_b = [&](int s) { return bar0 + 8 * (2 * F4_SP + s); };
    auto empty_b = [&](int s) { return bar0 + 8 * (2 * F4_SP + F4_SB + s); };
    auto full_a = [&](int s) { return bar0 + 8 * (2 * F4_SP + 2 * F4_SB + s); };
    auto empty_a = [&](int s) { return bar0 + 8 * (2 * F4_SP + 2 * F4_SB + F4_SA + s); };
    auto acc_full = [&](int a) { return bar0 + 8 * (2 * F4_SP + 2 * F4_SB + 2 * F4_SA + a); };
    auto acc_empty = [&](int a) { return bar0 + 8 * (2 * F4_SP + 2 * F4_SB + 2 * F4_SA + F4_NACC + a); };
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + F4_OFF_TMEM);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == F4_PROD) {
        if (lane == 0) {
            ptx::tma_prefetch(&tm_a);
            ptx::tma_prefetch(&tm_b);
            for (int s = 0; s < F4_SP; ++s) {
                ptx::mbar_init(full_p(s), 1);
                ptx::mbar_init(empty_p(s), 4);   // the 4 unpack warps, once per slot
            }
            for (int s = 0; s < F4_SB; ++s) {
                ptx::mbar_init(full_b(s), 1);
                ptx::mbar_init(empty_b(s), 1);
            }
            for (int s = 0; s < F4_SA; ++s) {
                ptx::mbar_init(full_a(s), 4);
                ptx::mbar_init(empty_a(s), 1);
            }
            for (int a = 0; a < F4_NACC; ++a) {
                ptx::mbar_init(acc_full(a), 1);
                ptx::mbar_init(acc_empty(a), 4);
            }
            ptx::fence_mbar_init();
        }
        __syncwarp();
        ptx::tmem_alloc(ptx::smem_u32(tmem_slot), 512);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp < 4) {   // block scales: every byte 2^1 (ue8m0 128), so D = sum (a/2 * 2)(v/2 * 2)
        uint32_t r[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = 0x80808080u;
        ptx::tmem_st_32x32b_x32(tmem + F4_SF_COL + ((uint32_t)(warp * 32) << 16), r);
        ptx::tmem_st_wait();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const int ntiles = fa.ntiles;

    if (warp == F4_PROD) {
        uint32_t gp = 0, gb = 0;   // packed slots / B stages issued
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            int tn, tm;
            f4_tile(fa, t, tn, tm);
            for (int s = 0; s < fa.nstages; ++s, ++gb) {
                if ((s & 1) == 0) {   // a packed slot = 2 stages of every activation row
                    const int ps = (int)(gp % F4_SP);
                    ptx::mbar_wait(empty_p(ps), ((gp / F4_SP) & 1u) ^ 1u);
                    if (lane == 0) {
                        ptx::mbar_arrive_expect_tx(full_p(ps), (uint32_t)F4_P_SLOT);
                        ptx::tma_load_2d(sbase + F4_OFF_P + ps * F4_P_SLOT, &tm_a, full_p(ps), s * (F4_KST / 4), tn * F4_BM);
                    }
                    __syncwarp();
                    ++gp;
                }
                const int bs = (int)(gb % F4_SB);
                ptx::mbar_wait(empty_b(bs), ((gb / F4_SB) & 1u) ^ 1u);
                if (lane == 0) {
                    ptx::mbar_arrive_expect_tx(full_b(bs), (uint32_t)F4_B_STAGE);
                    ptx::tma_load_2d(sbase + F4_OFF_B + bs * F4_B_STAGE, &tm_b, full_b(bs), s * (F4_KST / 2), tm * F4_BN);
                }
                __syncwarp();
            }
        }
    } else if (warp == F4_WAIT) {
        uint32_t g = 0, tl = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
            ptx::mbar_wait(acc_empty(tl % F4_NACC), ((tl / F4_NACC) & 1u) ^ 1u);
            for (int s = 0; s < fa.nstages; ++s, ++g) {
                ptx::mbar_wait(full_a(g % F4_SA), (g / F4_SA) & 1u);
                ptx::mbar_wait(full_b(g % F4_SB), (g / F4_SB) & 1u);
                ptx::named_bar_sync(F4_HANDOFF_BAR, 64);
            }
        }
    } else if (warp == F4_MMA) {
        constexpr uint32_t idesc = idesc_mxf4(F4_BM, F4_BN);
        const uint32_t sfa = tmem + F4_SF_COL, sfb = tmem + F4_SF_COL + 16;
        uint32_t g = 0, tl = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
            const uint32_t dt = tmem + (tl % F4_NACC) * F4_BN;
            for (int s = 0; s < fa.nstages; ++s, ++g) {
                const int sa = (int)(g % F4_SA), bs = (int)(g % F4_SB);
                ptx::named_bar_sync(F4_HANDOFF_BAR, 64);
                ptx::tc_fence_after();
                const uint64_t ad = ptx::desc_k_sw128(sbase + F4_OFF_A + sa * F4_A_STAGE);
                const uint64_t bd = ptx::desc_k_sw128(sbase + F4_OFF_B + bs * F4_B_STAGE);
                const int nk = s < fa.nstages - 1 ? 4 : fa.last_ksteps;
                for (int k = 0; k < nk; ++k)   // k-step = 64 codes = 32 bytes of every row (+2 in 16-byte units)
                    mma_mxf4_warp(dt, ad + 2 * k, bd + 2 * k, idesc, (s > 0 || k > 0) ? 1u : 0u, sfa, sfb);
                ptx::mma_commit_warp(empty_a(sa));
                ptx::mma_commit_warp(empty_b(bs));
                if (s == fa.nstages - 1) ptx::mma_commit_warp(acc_full(tl % F4_NACC));
                __syncwarp();
            }
        }
    } else if (warp >= F4_UNP0) {
        // thread = activation row r of the tile; each 16-byte packed chunk (64 codes) becomes two
        // 16-byte e2m1 chunks: word x -> (x & 0x33333333, (x >> 2) & 0x33333333)
        const int r = (warp - F4_UNP0) * 32 + lane;
        uint32_t g = 0, gp = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            for (int s = 0; s < fa.nstages; ++s, ++g) {
                const int ps = (int)(gp % F4_SP), sub = s & 1;
                if (sub == 0) ptx::mbar_wait(full_p(ps), (gp / F4_SP) & 1u);
                const uint32_t pbase = sbase + F4_OFF_P + ps * F4_P_SLOT;
                uint4 v[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {   // SW128 slot: 16-byte unit XOR row bits
                    const uint32_t lin = (uint32_t)(r * 128 + sub * 64 + 16 * c);
                    v[c] = ptx::lds128(pbase + (lin ^ (((lin >> 7) & 7u) << 4)));
                }
                uint32_t e[32];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const uint32_t w[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        e[8 * c + 2 * i] = w[i] & 0x33333333u;
                        e[8 * c + 2 * i + 1] = (w[i] >> 2) & 0x33333333u;
                    }
                }
                // release the slot only after its loaded values are used (an mbarrier arrive does not
                // wait for outstanding shared-memory loads; the refilling TMA could overtake them)
                if (sub == 1 || s == fa.nstages - 1) {
                    ptx::release_after_loads(empty_p(ps), 1u, v[0].x ^ v[1].x ^ v[2].x ^ v[3].x);
                    ++gp;
                }
                const int sa = (int)(g % F4_SA);
                ptx::mbar_wait(empty_a(sa), ((g / F4_SA) & 1u) ^ 1u);
                // SW128 K-major A stage: row r at (r/8)*1024 + (r%8)*128, 16-byte chunk j at (j ^ (r%8))*16
                const uint32_t row = sbase + F4_OFF_A + sa * F4_A_STAGE + (uint32_t)((r >> 3) * 1024 + (r & 7) * 128);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(row + (uint32_t)(((j ^ (r & 7)) << 4))),
                                 "r"(e[4 * j]), "r"(e[4 * j + 1]), "r"(e[4 * j + 2]), "r"(e[4 * j + 3])
                                 : "memory");
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(full_a(sa));
            }
        }
    } else {
        // ---------------- epilogue: D[n][m] fp32 (integer valued, |v| < 2^22) -> int32 C[m][n]
        const int quarter = warp;
        uint32_t tl = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
            int tn, tm;
            f4_tile(fa, t, tn, tm);
            const int64_t n = (int64_t)tn * F4_BM + quarter * 32 + lane;
            const int64_t m0 = (int64_t)tm * F4_BN;
            const uint32_t acc = tl % F4_NACC;
            ptx::mbar_wait(acc_full(acc), (tl / F4_NACC) & 1u);
            ptx::tc_fence_after();
            const uint32_t trow = tmem + acc * F4_BN + ((uint32_t)(quarter * 32) << 16);
            constexpr int NCH = (F4_BN + 31) / 32;   // (columns >= F4_BN of the last chunk are not stored)
#pragma unroll 1
            for (int c = 0; c < NCH; c += 2) {
                uint32_t r0[32], r1[32];
                ptx::tmem_ld_32x32b_x32(trow + c * 32, r0);
                ptx::tmem_ld_32x32b_x32(trow + c * 32 + 32, r1);
                ptx::tmem_ld_wait();
                if (c + 2 >= NCH) {   // the accumulator buffer is free again
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(acc_empty(acc));
                }
                if (n < fa.N) {
                    int32_t *cp = fa.C + (m0 + c * 32) * fa.ldc + n;
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (c * 32 + j < F4_BN && m0 + c * 32 + j < fa.M)
                            cp[(int64_t)j * fa.ldc] = __float_as_int(__uint_as_float(r0[j]) + 12582912.0f) - 0x4B400000;
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (c * 32 + 32 + j < F4_BN && m0 + c * 32 + 32 + j < fa.M)
                            cp[(int64_t)(32 + j) * fa.ldc] = __float_as_int(__uint_as_float(r1[j]) + 12582912.0f) - 0x4B400000;
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == F4_PROD) ptx::tmem_dealloc(tmem, 512);
}

// ---- weight expansion: packed codes -> e2m1 nibbles of level/2, in the unpack order (per 16 codes:
// nibbles 0-7 = codes 0,2,..,14, nibbles 8-15 = codes 1,3,..,15), 0 for k >= K.  One thread per
// 16-byte packed chunk (64 codes -> 32 bytes).
__global__ void expand_f4_kernel(const uint8_t *__restrict__ packed, int64_t rows, int64_t K, int64_t ld,
                                 uint32_t nib_tab, uint8_t *__restrict__ out, int64_t ld4) {
    const int64_t chunks = ld4 / 32;
    const int64_t total = rows * chunks;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / chunks, c = i - r * chunks;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (c * 16 + 16 <= ld) v = __ldg(reinterpret_cast<const uint4 *>(packed + r * ld + c * 16));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
        uint32_t o[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int64_t k0 = c * 64 + 16 * j + 2 * q;   // codes 2q and 2q+1 of word j
                const uint32_t c0 = (w[j] >> (4 * q)) & 3u, c1 = (w[j] >> (4 * q + 2)) & 3u;
                lo |= (k0 < K ? (nib_tab >> (4 * c0)) & 15u : 0u) << (4 * q);
                hi |= (k0 + 1 < K ? (nib_tab >> (4 * c1)) & 15u : 0u) << (4 * q);
            }
            o[2 * j] = lo;
            o[2 * j + 1] = hi;
        }
        uint4 *dst = reinterpret_cast<uint4 *>(out + r * ld4 + c * 32);
        dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
        dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
    }
}

typedef CUresult (*EncodeTiledF4)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool map_f4(CUtensorMap *m, const void *base, int64_t ld, int64_t rows, int box_rows) {
    static EncodeTiledF4 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledF4>(p);
    }
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld};
    cuuint32_t box[2] = {128u, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int64_t expand_f4_ld(int64_t K) { return (K + F4_KST - 1) / F4_KST * (F4_KST / 2); }

// e2m1 nibble of v/2 for an integer level v, or -1 if v/2 is not an e2m1 value
int f4_nibble_half(int32_t v) {
    static const int mag2[8] = {0, 1, 2, 3, 4, 6, 8, 12};   // 2 x {0, .5, 1, 1.5, 2, 3, 4, 6}
    const int a = v < 0 ? -v : v;
    for (int i = 0; i < 8; ++i)
        if (mag2[i] == a) return (v < 0 && a ? 8 : 0) | i;
    return -1;
}

dg_status expand_operand_f4(const uint8_t *packed, int64_t rows, int64_t K, int64_t ld, const int32_t levels[4],
                            uint8_t *out, int64_t ld4, cudaStream_t st) {
    uint32_t tab = 0;
    for (int c = 0; c < 4; ++c) {
        const int nb = f4_nibble_half(levels[c]);
        if (nb < 0) return DG_ERR_UNSUPPORTED;
        tab |= (uint32_t)nb << (4 * c);
    }
    if (rows == 0) return DG_OK;
    const int64_t work = rows * (ld4 / 32);
    int64_t blocks = (work + 255) / 256;
    if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
    expand_f4_kernel<<<(int)blocks, 256, 0, st>>>(packed, rows, K, ld, tab, out, ld4);
    return launch_status();
}

dg_status lut_gemm_f4(const uint8_t *At, int64_t lda, const uint8_t *W4, int64_t ld4, int64_t M, int64_t N, int64_t K,
                      int32_t *C, int64_t ldc, cudaStream_t st) {
    F4Args fa{};
    fa.M = M;
    fa.N = N;
    fa.ldc = ldc;
    fa.C = C;
    fa.nstages = (int32_t)((K + F4_KST - 1) / F4_KST);
    fa.last_ksteps = (int32_t)(((K - (int64_t)(fa.nstages - 1) * F4_KST) + 63) / 64);
    fa.ntn = (int32_t)((N + F4_BM - 1) / F4_BM);
    fa.ntm = (int32_t)((M + F4_BN - 1) / F4_BN);
    const int64_t ntiles = (int64_t)fa.ntn * fa.ntm;
    if (ntiles > INT32_MAX) return DG_ERR_SHAPE;
    fa.ntiles = (int32_t)ntiles;
    CUtensorMap ma, mb;
    if (!map_f4(&ma, At, lda, N, F4_BM) || !map_f4(&mb, W4, ld4, M, F4_BN)) return DG_ERR_CUDA;
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(lut_gemm_f4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, F4_ALLOC) != cudaSuccess)
            return DG_ERR_CUDA;
        attr = true;
    }
    const int grid = (int)(ntiles < num_sms() ? ntiles : num_sms());
    lut_gemm_f4_kernel<<<grid, F4_NT, F4_ALLOC, st>>>(ma, mb, fa);
    set_last_kernel("f4 gemm");
    return launch_status();
}

}  // namespace dg
