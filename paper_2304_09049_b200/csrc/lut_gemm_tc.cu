// lut_gemm_tc.cu — S5/S6/S7 on the 5th-gen tensor cores: the LUT-16 GEMM for PRODUCT
// tables (T[(p<<2)|q] = pl[p]*ql[q], dg_build_lut), as an unpack-to-int8 tcgen05 kind::i8
// GEMM.  Exact: every product and partial sum is an integer, accumulated in s32 TMEM.
//
//   D[p][q] = sum_{k<K} pl[P[p][k]] * ql[Q[q][k]]  ==  sum_k T[(P<<2)|Q]   (Alg. 1)
//
// Per CTA: one BM x BN output tile (BM = 128 TMEM lanes = rows of P, BN = 64/128/256 rows of Q).
// Warp roles (192 threads):
//   warp 0      TMA producer: packed 2-bit tiles [rows][32 B] (= 128 codes) -> packed smem ring
//   warp 1      MMA issuer (one thread): 4 x tcgen05.mma.kind::i8 (K=32) per 128-code stage
//   warps 2..5  unpackers, then epilogue: packed smem -> int8 levels via PRMT level lookup
//               (the paper's unpack step, P:123 / Alg. 1 line 9, producing levels instead of
//               indices) written in the UMMA K-major SWIZZLE_128B layout; after the K loop
//               they drain TMEM (tcgen05.ld) and apply the exact K-padding correction and the
//               optional fused requant (S7).
// The PRMT unpack emits the 16 codes of a 32-bit word in the order 0,2,4,6,8,..,1,3,..; the
// same permutation is applied to both operands, so the dot product is unchanged.
#include <cuda.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace dg {
namespace {

constexpr int BM = 128;        // TMEM lanes / P rows per tile
constexpr int KS = 128;        // codes per pipeline stage (one 128-byte SW128 row of int8)
constexpr int PKB = KS / 4;    // packed bytes per row per stage
constexpr int SP = 4;          // packed ring depth
constexpr int SU = 2;          // unpacked (int8) ring depth
constexpr int NT = 192;

template <int BN>
struct Layout {
    static constexpr int UNP_P = BM * KS;          // bytes per unpacked P stage
    static constexpr int UNP_Q = BN * KS;
    static constexpr int PK_P = BM * PKB;
    static constexpr int PK_Q = BN * PKB;
    static constexpr int OFF_UP = 0;
    static constexpr int OFF_UQ = OFF_UP + SU * UNP_P;
    static constexpr int OFF_PP = OFF_UQ + SU * UNP_Q;
    static constexpr int OFF_PQ = OFF_PP + SP * PK_P;
    static constexpr int OFF_BAR = OFF_PQ + SP * PK_Q;
    static constexpr int NBAR = 2 * SP + 2 * SU + 1;
    static constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
    static constexpr int BYTES = OFF_TMEM + 16;
    static constexpr int ALLOC = BYTES + 1024;     // slack for 1024-byte alignment
};

DG_DEV uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

// 16 packed codes -> 16 int8 levels (order 0,2,4,6 | 8,10,12,14 | 1,3,5,7 | 9,11,13,15)
DG_DEV uint4 unpack16(uint32_t x, uint32_t L) {
    const uint32_t X = x & 0x33333333u, Y = (x >> 2) & 0x33333333u;
    return make_uint4(prmt(L, L, X), prmt(L, L, X >> 16), prmt(L, L, Y), prmt(L, L, Y >> 16));
}

template <int BN>
__global__ void __launch_bounds__(NT, 1)
lut_gemm_tc_kernel(const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_q,
                   int64_t np, int64_t nq, int32_t nstages, uint32_t lp, uint32_t lq, int64_t corr,
                   void *__restrict__ D, int64_t ldd, RequantArgs rq, int has_rq) {
    using Lt = Layout<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = ptx::smem_u32(smem);
    const uint32_t bar0 = sbase + Lt::OFF_BAR;
    auto full_p = [&](int s) { return bar0 + 8 * s; };
    auto empty_p = [&](int s) { return bar0 + 8 * (SP + s); };
    auto full_u = [&](int s) { return bar0 + 8 * (2 * SP + s); };
    auto empty_u = [&](int s) { return bar0 + 8 * (2 * SP + SU + s); };
    const uint32_t acc_full = bar0 + 8 * (2 * SP + 2 * SU);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + Lt::OFF_TMEM);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t p0 = (int64_t)blockIdx.x * BM, q0 = (int64_t)blockIdx.y * BN;

    if (warp == 0) {
        if (lane == 0) {
            ptx::tma_prefetch(&tm_p);
            ptx::tma_prefetch(&tm_q);
            for (int s = 0; s < SP; ++s) {
                ptx::mbar_init(full_p(s), 1);
                ptx::mbar_init(empty_p(s), 4);
            }
            for (int s = 0; s < SU; ++s) {
                ptx::mbar_init(full_u(s), 4);
                ptx::mbar_init(empty_u(s), 1);
            }
            ptx::mbar_init(acc_full, 1);
            ptx::fence_mbar_init();
        }
        __syncwarp();
        ptx::tmem_alloc(ptx::smem_u32(tmem_slot), BN);   // BN int32 columns x 128 lanes
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer
        if (lane == 0) {
            for (int s = 0; s < nstages; ++s) {
                const int slot = s % SP;
                const uint32_t ph = (uint32_t)(s / SP) & 1u;
                ptx::mbar_wait(empty_p(slot), ph ^ 1u);
                ptx::mbar_arrive_expect_tx(full_p(slot), Lt::PK_P + Lt::PK_Q);
                ptx::tma_load_2d(sbase + Lt::OFF_PP + slot * Lt::PK_P, &tm_p, full_p(slot), s * PKB, (int32_t)p0);
                ptx::tma_load_2d(sbase + Lt::OFF_PQ + slot * Lt::PK_Q, &tm_q, full_p(slot), s * PKB, (int32_t)q0);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_i8(BM, BN);
            for (int s = 0; s < nstages; ++s) {
                const int slot = s % SU;
                const uint32_t ph = (uint32_t)(s / SU) & 1u;
                ptx::mbar_wait(full_u(slot), ph);
                ptx::tc_fence_after();
                const uint32_t a = sbase + Lt::OFF_UP + slot * Lt::UNP_P;
                const uint32_t b = sbase + Lt::OFF_UQ + slot * Lt::UNP_Q;
#pragma unroll
                for (int k = 0; k < KS / 32; ++k)
                    ptx::mma_i8_ss(tmem, ptx::desc_k_sw128(a + 32 * k), ptx::desc_k_sw128(b + 32 * k), idesc,
                                   (s > 0 || k > 0) ? 1u : 0u);
                ptx::mma_commit(empty_u(slot));
            }
            ptx::mma_commit(acc_full);
        }
    } else {
        // ---------------- unpackers (warps 2..5, 128 threads)
        const int ut = threadIdx.x - 64;
        constexpr int ITEMS = (BM + BN) * 2;   // 16-byte packed chunks per stage
        for (int s = 0; s < nstages; ++s) {
            const int sp = s % SP, su = s % SU;
            ptx::mbar_wait(full_p(sp), (uint32_t)(s / SP) & 1u);
            ptx::mbar_wait(empty_u(su), ((uint32_t)(s / SU) & 1u) ^ 1u);
            const uint8_t *pk_p = smem + Lt::OFF_PP + sp * Lt::PK_P;
            const uint8_t *pk_q = smem + Lt::OFF_PQ + sp * Lt::PK_Q;
            uint8_t *up = smem + Lt::OFF_UP + su * Lt::UNP_P;
            uint8_t *uq = smem + Lt::OFF_UQ + su * Lt::UNP_Q;
#pragma unroll 2
            for (int it = ut; it < ITEMS; it += 128) {
                const int row = it >> 1, h = it & 1;
                const bool isp = row < BM;
                const int r = isp ? row : row - BM;
                const uint4 v = *reinterpret_cast<const uint4 *>((isp ? pk_p : pk_q) + r * PKB + h * 16);
                const uint32_t L = isp ? lp : lq;
                uint8_t *dst = (isp ? up : uq) + (r >> 3) * 1024 + (r & 7) * 128;
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int chunk = (h * 4 + j) ^ (r & 7);
                    *reinterpret_cast<uint4 *>(dst + chunk * 16) = unpack16(w[j], L);
                }
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(empty_p(sp));
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(full_u(su));
        }

        // ---------------- epilogue: TMEM -> registers -> global
        ptx::mbar_wait(acc_full, 0);
        ptx::tc_fence_after();
        const int quarter = warp & 3;
        const int64_t p = p0 + quarter * 32 + lane;
        const uint32_t trow = tmem + ((uint32_t)(quarter * 32) << 16);
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            ptx::tmem_ld_32x32b_x32(trow + c * 32, r);
            ptx::tmem_ld_wait();
            const int64_t qc = q0 + c * 32;
            if (p >= np || qc >= nq) continue;
            int32_t v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = (int32_t)((int64_t)(int32_t)r[j] - corr);
            if (!has_rq) {
                int32_t *dp = reinterpret_cast<int32_t *>(D) + p * ldd + qc;
                if (qc + 32 <= nq && (ldd & 3) == 0 && ((reinterpret_cast<uintptr_t>(D) & 15) == 0)) {
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        *reinterpret_cast<int4 *>(dp + j) = make_int4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                } else {
                    for (int j = 0; j < 32; ++j)
                        if (qc + j < nq) dp[j] = v[j];
                }
            } else {
                uint32_t o[2] = {0, 0};
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (qc + j < nq) o[j >> 4] |= requant_one(rq, v[j], p, qc + j) << (2 * (j & 15));
                uint8_t *dp = reinterpret_cast<uint8_t *>(D) + p * ldd + (qc >> 2);
                const int nbytes = (int)((nq - qc) >= 32 ? 8 : ((nq - qc) + 3) / 4);
                if (nbytes == 8 && ((reinterpret_cast<uintptr_t>(dp) & 7) == 0)) {
                    *reinterpret_cast<uint2 *>(dp) = make_uint2(o[0], o[1]);
                } else {
                    for (int b = 0; b < nbytes; ++b) dp[b] = (uint8_t)(o[b >> 2] >> (8 * (b & 3)));
                }
            }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, BN);
}

// ---------------------------------------------------------------- host
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

bool make_map(CUtensorMap *m, const uint8_t *base, int64_t ld, int64_t rows, int box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld};
    cuuint32_t box[2] = {(cuuint32_t)PKB, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

uint32_t pack_levels(const int32_t l[4]) {
    uint32_t L = 0;
    for (int i = 0; i < 4; ++i) L |= ((uint32_t)(l[i] & 0xFF)) << (8 * i);
    return L;
}

template <int BN>
dg_status launch(const uint8_t *P, int64_t ldp, const uint8_t *Q, int64_t ldq, int64_t np, int64_t nq, int64_t K,
                 const int32_t pl[4], const int32_t ql[4], void *D, int64_t ldd, const RequantArgs *rq,
                 cudaStream_t st) {
    CUtensorMap mp, mq;
    if (!make_map(&mp, P, ldp, np, BM) || !make_map(&mq, Q, ldq, nq, BN)) return DG_ERR_CUDA;
    const int32_t nstages = (int32_t)((K + KS - 1) / KS);
    const int64_t Kp = (int64_t)nstages * KS;
    const int64_t corr = (Kp - K) * (int64_t)pl[0] * (int64_t)ql[0];
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(lut_gemm_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Layout<BN>::ALLOC) != cudaSuccess)
            return DG_ERR_CUDA;
        attr_set = true;
    }
    RequantArgs dummy{};
    dim3 grid((unsigned)((np + BM - 1) / BM), (unsigned)((nq + BN - 1) / BN));
    if (grid.y > 65535) return DG_ERR_SHAPE;
    lut_gemm_tc_kernel<BN><<<grid, NT, Layout<BN>::ALLOC, st>>>(mp, mq, np, nq, nstages, pack_levels(pl),
                                                                 pack_levels(ql), corr, D, ldd,
                                                                 rq ? *rq : dummy, rq ? 1 : 0);
    return launch_status();
}

}  // namespace

bool tc_available() {
    static int ok = -1;
    if (ok < 0) {
        int dev = 0, major = 0, minor = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
        ok = (major == 10 && minor == 0 && encode_fn() != nullptr) ? 1 : 0;
    }
    return ok == 1;
}

dg_status lut_gemm_tc(const uint8_t *P, int64_t ldp, const uint8_t *Q, int64_t ldq, int64_t np, int64_t nq,
                      int64_t K, const int32_t pl[4], const int32_t ql[4], void *D, int64_t ldd,
                      const RequantArgs *rq, cudaStream_t st) {
    if (np > ((int64_t)1 << 31) - 1 || nq > ((int64_t)1 << 31) - 1) return DG_ERR_SHAPE;
    if (nq > 128) return launch<256>(P, ldp, Q, ldq, np, nq, K, pl, ql, D, ldd, rq, st);
    if (nq > 64) return launch<128>(P, ldp, Q, ldq, np, nq, K, pl, ql, D, ldd, rq, st);
    return launch<64>(P, ldp, Q, ldq, np, nq, K, pl, ql, D, ldd, rq, st);
}

}  // namespace dg
