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
#include <string.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace dg {
namespace {

constexpr int BM = 128;        // TMEM lanes / P rows per tile
constexpr int KS = 128;        // codes per unpacked stage (one 128-byte SW128 row of int8)
constexpr int PKB = KS / 4;    // packed bytes per row per unpacked stage
constexpr int PKS_MAX = 128;   // packed bytes per row per packed (TMA / bulk) stage: up to 4 unpacked stages
constexpr int NUM_UNPACK_WARPS = 6;
constexpr int NUM_UGROUPS = 2;         // unpack groups own alternate stages (in order within a group)
constexpr int UGROUP_WARPS = NUM_UNPACK_WARPS / NUM_UGROUPS;
constexpr int NUM_EPI_WARPS = 8;       // 2 per TMEM lane quarter, each owning half the columns
constexpr int UNPACK_WARP0 = 2;
constexpr int EPI_WARP0 = UNPACK_WARP0 + NUM_UNPACK_WARPS;
constexpr int NT = 32 * (EPI_WARP0 + NUM_EPI_WARPS);   // 448 threads

template <int BN>
struct Cfg {
    // Ring depths are multiples of NUM_UGROUPS so that a group, which consumes its stages in
    // order, can never run a full phase ahead on a slot (mbarrier parity aliasing).
    static constexpr int SU = BN == 256 ? 2 : 4;            // unpacked (int8) ring depth
    static constexpr int SP = BN == 256 ? 2 : (BN == 128 ? 2 : 4);  // packed ring depth (128 B/row stages)
    static constexpr int UNP_P = BM * KS;                  // bytes per unpacked P stage
    static constexpr int UNP_Q = BN * KS;
    static constexpr int PK_P = BM * PKS_MAX;
    static constexpr int PK_Q = BN * PKS_MAX;
    static constexpr int OFF_UP = 0;
    static constexpr int OFF_UQ = OFF_UP + SU * UNP_P;
    static constexpr int OFF_PP = OFF_UQ + SU * UNP_Q;
    static constexpr int OFF_PQ = OFF_PP + SP * PK_P;
    static constexpr int OFF_BAR = OFF_PQ + SP * PK_Q;
    static constexpr int NACC = BN == 256 ? 2 : 4;          // TMEM accumulator buffers
    static constexpr int NBAR = 2 * SP + 2 * SU + 2 * NACC;
    static constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
    static constexpr int BYTES = OFF_TMEM + 16;
    static constexpr int ALLOC = BYTES + 1024;             // slack for 1024-byte alignment
    static constexpr int TMEM_COLS = NACC * BN;            // multi-buffered accumulator (<= 512)
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

#ifdef DG_TRACE
// Debug timeline (compile with -DDG_TRACE): CTA 0 records %globaltimer at pipeline events.
__device__ unsigned long long *g_dg_trace = nullptr;
DG_DEV unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define DG_TR(ev, idx)                                                                 \
    do {                                                                               \
        if (g_dg_trace && blockIdx.x == 0 && (idx) < 64) g_dg_trace[(ev) * 64 + (idx)] = gtimer(); \
    } while (0)
#else
#define DG_TR(ev, idx) \
    do {               \
    } while (0)
#endif

struct TileArgs {
    int64_t np, nq;
    int32_t nstages;       // K stages of 128 codes
    int32_t last_ksteps;   // MMA k-steps (32 codes) issued in the last stage: 1..4
    int32_t ntp, ntq;      // tiles along P and Q
    uint32_t lp, lq;       // int8 level tables of P / Q codes (4 bytes)
    int64_t corr;          // exact correction for codes in [K, K_mma): (K_mma-K)*pl[0]*ql[0]
    void *D;
    int64_t ldd;
    int32_t has_rq;
    int32_t fast_rq;       // requant with at most a bias: int32 threshold compares
    int32_t thr[3];        // int32 thresholds on acc_raw + bias (K-pad correction folded in)
    int32_t dir;
    int32_t pks;           // packed bytes per row per packed stage (smem row pitch), <= 128
    int32_t nps;           // packed stages per tile
    int32_t bulk;          // 1: each packed stage is one contiguous tile -> cp.async.bulk
    const uint8_t *P, *Q;  // operand bases (bulk mode)
    int64_t ldp, ldq;
};

DG_DEV void store_codes32(uint8_t *dp, uint32_t o0, uint32_t o1, int nbytes) {
#pragma unroll
    for (int b = 0; b < 8; ++b)
        if (b < nbytes) dp[b] = (uint8_t)((b < 4 ? o0 : o1) >> (8 * (b & 3)));
}

// Epilogue for one 32-column chunk of row p: int32 output, or requant with residuals /
// partial chunks.  Kept out of line so the hot requant loop stays small in the I-cache.
__device__ __noinline__ void epilogue_general(const TileArgs &ta, const RequantArgs &rq, uint32_t taddr,
                                              int64_t p, int64_t qc) {
    uint32_t rr[32];
    ptx::tmem_ld_32x32b_x32(taddr, rr);
    ptx::tmem_ld_wait();
    if (p >= ta.np || qc >= ta.nq) return;
    int32_t v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = (int32_t)rr[j] - (int32_t)ta.corr;
    if (!ta.has_rq) {
        int32_t *dp = reinterpret_cast<int32_t *>(ta.D) + p * ta.ldd + qc;
        if (qc + 32 <= ta.nq && (ta.ldd & 3) == 0 && ((reinterpret_cast<uintptr_t>(ta.D) & 15) == 0)) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<int4 *>(dp + j) = make_int4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
            for (int j = 0; j < 32; ++j)
                if (qc + j < ta.nq) dp[j] = v[j];
        }
        return;
    }
    uint8_t *dp = reinterpret_cast<uint8_t *>(ta.D) + p * ta.ldd + (qc >> 2);
    if (qc + 32 <= ta.nq) {
        const uint2 o = requant_row32(rq, v, p, qc);
        if ((reinterpret_cast<uintptr_t>(dp) & 7) == 0) *reinterpret_cast<uint2 *>(dp) = o;
        else store_codes32(dp, o.x, o.y, 8);
        return;
    }
    uint32_t o0 = 0, o1 = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        if (qc + j < ta.nq) {
            const uint32_t cd = requant_one(rq, v[j], p, qc + j);
            if (j < 16) o0 |= cd << (2 * j);
            else o1 |= cd << (2 * (j - 16));
        }
    }
    store_codes32(dp, o0, o1, (int)((ta.nq - qc + 3) / 4));
}

// Persistent warp-specialised kernel, one CTA per SM.
//   warp 0: TMA producer   warp 1: MMA issuer   warps 2..9: unpack   warps 10..13: epilogue
template <int BN>
__global__ void __launch_bounds__(NT, 1)
lut_gemm_tc_kernel(const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_q,
                   const __grid_constant__ TileArgs ta,
                   const __grid_constant__ RequantArgs rq) {
    using C = Cfg<BN>;
    constexpr int SP = C::SP, SU = C::SU;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = ptx::smem_u32(smem);
    const uint32_t bar0 = sbase + C::OFF_BAR;
    auto full_p = [&](int s) { return bar0 + 8 * s; };
    auto empty_p = [&](int s) { return bar0 + 8 * (SP + s); };
    auto full_u = [&](int s) { return bar0 + 8 * (2 * SP + s); };
    auto empty_u = [&](int s) { return bar0 + 8 * (2 * SP + SU + s); };
    constexpr int NACC = C::NACC;
    auto acc_full = [&](int a) { return bar0 + 8 * (2 * SP + 2 * SU + a); };
    auto acc_empty = [&](int a) { return bar0 + 8 * (2 * SP + 2 * SU + NACC + a); };
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + C::OFF_TMEM);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = ta.ntp * ta.ntq;

    if (warp == 0) {
        if (lane == 0) {
            ptx::tma_prefetch(&tm_p);
            ptx::tma_prefetch(&tm_q);
            for (int s = 0; s < SP; ++s) {
                ptx::mbar_init(full_p(s), 1);
                ptx::mbar_init(empty_p(s), (PKS_MAX / PKB) * UGROUP_WARPS);   // per sub-stage, per warp
            }
            for (int s = 0; s < SU; ++s) {
                ptx::mbar_init(full_u(s), UGROUP_WARPS);     // the warps of the owning group
                ptx::mbar_init(empty_u(s), 1);
            }
            for (int a = 0; a < NACC; ++a) {
                ptx::mbar_init(acc_full(a), 1);
                ptx::mbar_init(acc_empty(a), NUM_EPI_WARPS);
            }
            ptx::fence_mbar_init();
        }
        __syncwarp();
        ptx::tmem_alloc(ptx::smem_u32(tmem_slot), C::TMEM_COLS);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- producer: packed 2-bit tiles (TMA 2-D boxes, or 1-D bulk copies when the
        // whole K extent of a tile is contiguous)
        if (lane == 0) {
            uint32_t g = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int64_t p0 = (int64_t)(t / ta.ntq) * BM, q0 = (int64_t)(t % ta.ntq) * BN;
                for (int s = 0; s < ta.nps; ++s, ++g) {
                    const int slot = g % SP;
                    ptx::mbar_wait(empty_p(slot), ((g / SP) & 1u) ^ 1u);
                    DG_TR(0, g);
                    const uint32_t dp = sbase + C::OFF_PP + slot * C::PK_P, dq = sbase + C::OFF_PQ + slot * C::PK_Q;
                    if (ta.bulk) {
                        const int64_t rp = ta.np - p0 < BM ? ta.np - p0 : BM, rq_ = ta.nq - q0 < BN ? ta.nq - q0 : BN;
                        const uint32_t bp = (uint32_t)(rp * ta.ldp), bq = (uint32_t)(rq_ * ta.ldq);
                        ptx::mbar_arrive_expect_tx(full_p(slot), bp + bq);
                        ptx::bulk_load(dp, ta.P + p0 * ta.ldp, bp, full_p(slot));
                        ptx::bulk_load(dq, ta.Q + q0 * ta.ldq, bq, full_p(slot));
                    } else {
                        ptx::mbar_arrive_expect_tx(full_p(slot), (uint32_t)((BM + BN) * ta.pks));
                        ptx::tma_load_2d(dp, &tm_p, full_p(slot), s * ta.pks, (int32_t)p0);
                        ptx::tma_load_2d(dq, &tm_q, full_p(slot), s * ta.pks, (int32_t)q0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (whole warp; one lane elected inside the *_warp helpers)
        {
            constexpr uint32_t idesc = ptx::idesc_i8(BM, BN);
            uint32_t g = 0, tl = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
                const uint32_t acc = tl % NACC;
                ptx::mbar_wait(acc_empty(acc), ((tl / NACC) & 1u) ^ 1u);
                DG_TR(1, tl);
                ptx::tc_fence_after();
                const uint32_t dt = tmem + acc * BN;
                for (int s = 0; s < ta.nstages; ++s, ++g) {
                    const int slot = g % SU;
                    ptx::mbar_wait(full_u(slot), (g / SU) & 1u);
                    DG_TR(2, g);
                    ptx::tc_fence_after();
                    const uint32_t a = sbase + C::OFF_UP + slot * C::UNP_P;
                    const uint32_t b = sbase + C::OFF_UQ + slot * C::UNP_Q;
                    const int ksteps = (s == ta.nstages - 1) ? ta.last_ksteps : KS / 32;
#pragma unroll
                    for (int k = 0; k < KS / 32; ++k)
                        if (k < ksteps)
                            ptx::mma_i8_ss_warp(dt, ptx::desc_k_sw128(a + 32 * k), ptx::desc_k_sw128(b + 32 * k), idesc,
                                                (s > 0 || k > 0) ? 1u : 0u);
                    ptx::mma_commit_warp(empty_u(slot));
                }
                ptx::mma_commit_warp(acc_full(acc));
            }
        }
    } else if (warp < EPI_WARP0) {
        // ---------------- unpackers: packed smem -> int8 levels in the SW128 K-major layout.
        // Group j (UGROUP_WARPS warps) owns unpacked stages g = j, j + NUM_UGROUPS, ... so that
        // NUM_UGROUPS stages are in flight and the per-stage handoff latency overlaps.
        const int uw = warp - UNPACK_WARP0;
        const int grp = uw / UGROUP_WARPS, gt = (uw % UGROUP_WARPS) * 32 + lane;
        constexpr int ITEMS = (BM + BN) * 2;     // 16-byte packed chunks (64 codes) per unpacked stage
        const int nsub = (ta.pks + PKB - 1) / PKB;
        uint32_t g = 0, gp = 0;                  // global unpacked / packed stage counters
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            for (int s = 0; s < ta.nstages; ++s, ++g) {
                const int sub = s % nsub;
                const bool last_sub = sub == nsub - 1 || s == ta.nstages - 1;
                const uint32_t my_gp = gp;
                if (last_sub) ++gp;
                if ((int)(g % NUM_UGROUPS) != grp) continue;
                const int sp = my_gp % SP, su = g % SU;
                // 16-byte chunk h covers MMA k-steps 2h, 2h+1: skip chunks no MMA reads
                const int hmax = (s == ta.nstages - 1) ? (ta.last_ksteps + 1) / 2 : 2;
                ptx::mbar_wait(full_p(sp), (my_gp / SP) & 1u);
                if (gt == 0) DG_TR(3, g);
                ptx::mbar_wait(empty_u(su), ((g / SU) & 1u) ^ 1u);
                if (gt == 0) DG_TR(4, g);
                const uint8_t *pk_p = smem + C::OFF_PP + sp * C::PK_P;
                const uint8_t *pk_q = smem + C::OFF_PQ + sp * C::PK_Q;
                uint8_t *up = smem + C::OFF_UP + su * C::UNP_P;
                uint8_t *uq = smem + C::OFF_UQ + su * C::UNP_Q;
#pragma unroll 2
                for (int it = gt; it < ITEMS; it += 32 * UGROUP_WARPS) {
                    const int row = it >> 1, h = it & 1;
                    if (h >= hmax) continue;
                    const bool isp = row < BM;
                    const int r = isp ? row : row - BM;
                    // tensor mode: the TMA wrote 128-byte rows with the 128B swizzle (16-byte chunk
                    // index XOR row%8), which makes this column read conflict-free
                    const int cidx = ta.bulk ? (sub * 2 + h) : ((sub * 2 + h) ^ (r & 7));
                    const uint4 v = *reinterpret_cast<const uint4 *>((isp ? pk_p : pk_q) + r * ta.pks + cidx * 16);
                    const uint32_t L = isp ? ta.lp : ta.lq;
                    uint8_t *dst = (isp ? up : uq) + (r >> 3) * 1024 + (r & 7) * 128;
                    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int chunk = (h * 4 + j) ^ (r & 7);
                        *reinterpret_cast<uint4 *>(dst + chunk * 16) = unpack16(w[j], L);
                    }
                }
                if (gt == 0) DG_TR(9, g);
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (gt == 0) DG_TR(10, g);
                if (lane == 0) {
                    ptx::mbar_arrive(full_u(su));
                    // release the packed slot once per sub-stage; a short final packed stage
                    // releases the sub-stages it does not have as well
                    const int extra = (s == ta.nstages - 1) ? (PKS_MAX / PKB - 1 - sub) : (sub == nsub - 1 ? PKS_MAX / PKB - nsub : 0);
                    ptx::mbar_arrive(empty_p(sp));
                    for (int e = 0; e < extra; ++e) ptx::mbar_arrive(empty_p(sp));
                }
                if (gt == 0) DG_TR(5, g);
            }
        }
    } else {
        // ---------------- epilogue: TMEM -> registers -> (requant) -> global
        // 8 warps: lane quarter = warp % 4 (TMEM access rule), column half = (warp - EPI_WARP0) / 4
        constexpr int HALF = BN / 2, NCH = HALF / 32;
        const int quarter = warp & 3, half = (warp - EPI_WARP0) >> 2;
        const bool col_bias = rq.bias && rq.bias_axis == 0;
        uint32_t tl = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
            const uint32_t acc = tl % NACC;
            const int64_t p = (int64_t)(t / ta.ntq) * BM + quarter * 32 + lane;
            const int64_t q0 = (int64_t)(t % ta.ntq) * BN + half * HALF;
            ptx::mbar_wait(acc_full(acc), (tl / NACC) & 1u);
            if (warp == EPI_WARP0 && lane == 0) DG_TR(6, tl);
            ptx::tc_fence_after();
            const uint32_t trow = tmem + acc * BN + half * HALF + ((uint32_t)(quarter * 32) << 16);
            const bool fast = ta.fast_rq && q0 + HALF <= ta.nq;
            const int32_t rb = (fast && rq.bias && rq.bias_axis == 1 && p < ta.np) ? __ldg(rq.bias + p) : 0;
            if (!fast) {
                // int32 output / residual requant / ragged tail: out of line, reloads TMEM itself
#pragma unroll 1
                for (int c = 0; c < NCH; ++c) epilogue_general(ta, rq, trow + c * 32, p, q0 + c * 32);
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(acc_empty(acc));   // accumulator buffer drained
            } else {
                uint32_t r[2][32];
                ptx::tmem_ld_32x32b_x32(trow, r[0]);
#pragma unroll
                for (int c = 0; c < NCH; ++c) {
                    const int64_t qc = q0 + c * 32;
                    int4 bx[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j)   // warp-uniform bias loads, issued before the TMEM wait
                        bx[j] = col_bias ? __ldg(reinterpret_cast<const int4 *>(rq.bias + qc) + j) : make_int4(rb, rb, rb, rb);
                    ptx::tmem_ld_wait();
                    if (c + 1 < NCH) ptx::tmem_ld_32x32b_x32(trow + (c + 1) * 32, r[(c + 1) & 1]);
                    if (c == NCH - 1) {   // all of this warp's columns are in registers: free the buffer
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(acc_empty(acc));
                        if (warp == EPI_WARP0 && lane == 0) DG_TR(7, tl);
                    }
                    if (p >= ta.np) continue;
                    // v = acc_raw + bias; code = number of exact thresholds passed, counted from
                    // sign bits: (t - v) < 0 <=> v > t  (|t|, |v| < 2^30: no overflow)
                    uint32_t o0 = 0, o1 = 0;
                    if (ta.dir > 0) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int4 b4 = bx[j >> 2];
                            const int32_t b = (j & 3) == 0 ? b4.x : (j & 3) == 1 ? b4.y : (j & 3) == 2 ? b4.z : b4.w;
                            const int32_t v = (int32_t)r[c & 1][j];
                            const uint32_t cd = ((uint32_t)(ta.thr[0] - v - b) >> 31) + ((uint32_t)(ta.thr[1] - v - b) >> 31) +
                                                ((uint32_t)(ta.thr[2] - v - b) >> 31);
                            if (j < 16) o0 += cd << (2 * j);
                            else o1 += cd << (2 * (j - 16));
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int4 b4 = bx[j >> 2];
                            const int32_t b = (j & 3) == 0 ? b4.x : (j & 3) == 1 ? b4.y : (j & 3) == 2 ? b4.z : b4.w;
                            const int32_t v = (int32_t)r[c & 1][j];
                            const uint32_t cd = ((uint32_t)(v + b - ta.thr[0] - 1) >> 31) +
                                                ((uint32_t)(v + b - ta.thr[1] - 1) >> 31) +
                                                ((uint32_t)(v + b - ta.thr[2] - 1) >> 31);
                            if (j < 16) o0 += cd << (2 * j);
                            else o1 += cd << (2 * (j - 16));
                        }
                    }
                    uint8_t *dp = reinterpret_cast<uint8_t *>(ta.D) + p * ta.ldd + (qc >> 2);
                    if ((reinterpret_cast<uintptr_t>(dp) & 7) == 0) *reinterpret_cast<uint2 *>(dp) = make_uint2(o0, o1);
                    else store_codes32(dp, o0, o1, 8);
                }
            }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(tmem, C::TMEM_COLS);
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

bool make_map(CUtensorMap *m, const uint8_t *base, int64_t ld, int64_t rows, int box_rows, int box_inner) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld};
    cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, box_inner == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
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
    int64_t acc_bound = 0;   // K * max |pl[a] * ql[b]|
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
            const int64_t e = (int64_t)pl[a] * ql[b];
            acc_bound = (e < 0 ? -e : e) > acc_bound ? (e < 0 ? -e : e) : acc_bound;
        }
    acc_bound *= K;
    CUtensorMap mp, mq;
    memset(&mp, 0, sizeof(mp));
    memset(&mq, 0, sizeof(mq));
    // A packed stage carries up to 128 B (512 codes) of every row.  When both operands' rows fit
    // one packed stage and the row pitches match, each tile is one contiguous span -> bulk copy.
    // (only rows of <= 32 B: wider rows are read column-wise from smem and need the TMA swizzle)
    const bool bulk = ldp == ldq && ldp <= 32 && (((uintptr_t)P | (uintptr_t)Q) & 15) == 0;
    const int pks = bulk ? (int)ldp : PKS_MAX;
    if (!bulk && (!make_map(&mp, P, ldp, np, BM, pks) || !make_map(&mq, Q, ldq, nq, BN, pks))) return DG_ERR_CUDA;
    TileArgs ta{};
    ta.np = np;
    ta.nq = nq;
    ta.nstages = (int32_t)((K + KS - 1) / KS);
    const int64_t kmma = (K + 31) / 32 * 32;
    ta.last_ksteps = (int32_t)((kmma - (int64_t)(ta.nstages - 1) * KS) / 32);
    ta.ntp = (int32_t)((np + BM - 1) / BM);
    ta.ntq = (int32_t)((nq + BN - 1) / BN);
    ta.lp = pack_levels(pl);
    ta.lq = pack_levels(ql);
    ta.corr = (kmma - K) * (int64_t)pl[0] * (int64_t)ql[0];
    ta.D = D;
    ta.ldd = ldd;
    ta.pks = pks;
    ta.bulk = bulk ? 1 : 0;
    ta.P = P;
    ta.Q = Q;
    ta.ldp = ldp;
    ta.ldq = ldq;
    ta.nps = (int32_t)((ta.nstages + (pks + PKB - 1) / PKB - 1) / ((pks + PKB - 1) / PKB));
    ta.has_rq = rq ? 1 : 0;
    ta.fast_rq = 0;
    if (rq && !rq->res && !rq->res_codes && acc_bound < ((int64_t)1 << 29) &&
        (!rq->bias || rq->bias_axis == 1 || (((uintptr_t)rq->bias) & 15) == 0)) {
        // x = acc_raw + bias with acc_raw = acc + corr:  acc + bias >= t  <=>  x > t + corr - 1
        ta.fast_rq = 1;
        ta.dir = rq->dir;
        for (int j = 0; j < 3; ++j) {
            const int64_t t = rq->thr[j];
            int64_t u;
            if (t == INT64_MAX || t == INT64_MIN) u = t;   // never / always sentinels
            else u = rq->dir > 0 ? t + ta.corr - 1 : t + ta.corr;
            const int64_t LIM = (int64_t)1 << 30;          // |acc + bias| < 2^30 (dg.h)
            ta.thr[j] = (int32_t)(u > LIM ? LIM : (u < -LIM ? -LIM : u));
        }
    }
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(lut_gemm_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Cfg<BN>::ALLOC) != cudaSuccess)
            return DG_ERR_CUDA;
        attr_set = true;
    }
    RequantArgs dummy{};
    const int64_t ntiles = (int64_t)ta.ntp * ta.ntq;
    if (ntiles > INT32_MAX) return DG_ERR_SHAPE;
    const int grid = (int)(ntiles < num_sms() ? ntiles : num_sms());
    lut_gemm_tc_kernel<BN><<<grid, NT, Cfg<BN>::ALLOC, st>>>(mp, mq, ta, rq ? *rq : dummy);
    set_last_kernel(BN == 256 ? "tc_ss bn=256" : BN == 128 ? "tc_ss bn=128" : "tc_ss bn=64");
    return launch_status();
}

}  // namespace

#ifdef DG_TRACE
extern "C" __attribute__((visibility("default"))) int dg_debug_set_trace(void *dev_buf) {
    unsigned long long *p = (unsigned long long *)dev_buf;
    return cudaMemcpyToSymbol(g_dg_trace, &p, sizeof(p)) == cudaSuccess ? 0 : -1;
}
#endif

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
