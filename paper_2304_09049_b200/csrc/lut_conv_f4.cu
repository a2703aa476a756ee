// lut_conv_f4.cu — the LUT-16 convolution on the block-scaled FP4 tensor-core path (tcgen05
// kind::mxf4, e2m1 x e2m1; SURVEY §8(f) rank 2 on the conv workloads), in the conv orientation
//
//   out[pixel][co] = sum_{k<K} T[(w[co][k] << 2) | x_col[pixel][k]] = sum_k wl[w] * al[x]
//
// with the activation codes unpacked on chip (Alg. 1 line 9) into e2m1 nibbles (for activation
// levels al = {0,1,2,3} the 2-bit code c IS the e2m1 encoding of c/2: two nibble masks per 16
// codes), weights expanded offline to e2m1 nibbles of wl/2 (dg_expand_operand_f4), unit block
// scales 2 x 2, so the fp32 tensor-core sum is sum(wl*al) exactly (every partial sum is an integer
// below 2^22; the accumulators start at 1.5*2^23 so that the low 16 bits of an fp32 accumulator ARE
// the int16 of its integer value: the 16-bit SIMD requant of the int8 kernel reads them unchanged).
//
// Tile 128 pixels x 128 output channels, three fp32 accumulator buffers (384 TMEM columns) + 32
// block-scale columns.  Persistent, warp-specialised, one CTA per SM:
//   warps 0..3   epilogue (lane quarter = warp): TMEM -> requant (S7) or int32 -> NHWC output
//   warps 4..7   unpack: thread = output pixel; 1x1 convs read TMA slots of the NHWC tensor,
//                others gather their pixel's taps (implicit im2col, cp.async ring); -> e2m1 A stage
//   warp 8       producer: TMA of the e2m1 weight stages (and of the packed slots of direct convs)
//   warp 9       waiter: mbarrier waits, hands each stage to the MMA warp through a named barrier
//   warp 10      MMA issuer (whole warp, one lane elected inside the asm)
#include <cuda.h>
#include <stdio.h>
#include <string.h>

#include "common.cuh"
#include "requant16.cuh"
#include "tc_ptx.cuh"

namespace dg {
namespace {

constexpr int CF_BM = 128, CF_BN = 128;
constexpr int CF_KST = 256;                        // codes per stage: 128 bytes of e2m1 per row = 4 MMAs (K = 64)
constexpr int CF_NACC_MAX = 4, CF_SA_MAX = 6, CF_SB = 6, CF_SP = 3, CF_IG = 6;
constexpr int CF_A_STAGE = CF_BM * CF_KST / 2;     // 16 KB, SW128 K-major
constexpr int CF_B_STAGE = CF_BN * CF_KST / 2;     // 16 KB, SW128 K-major
constexpr int CF_P_SLOT = CF_BM * 128;             // 16 KB: 512 packed codes of every row (2 stages)
constexpr int CF_RING = CF_BM * 64;                // 8 KB: one stage (64 packed bytes) of every row
constexpr int CF_P_REGION = CF_SP * CF_P_SLOT > CF_IG * CF_RING ? CF_SP * CF_P_SLOT : CF_IG * CF_RING;
constexpr int CF_TAB_PAIRS = 1024;                 // per-column requant offsets: Cout <= 2048
constexpr int CF_OFF_B = 0;
constexpr int CF_OFF_A = CF_OFF_B + CF_SB * CF_B_STAGE;
constexpr int CF_OFF_P = CF_OFF_A + 4 * CF_A_STAGE;   // (shared-memory A: 4 stages)
constexpr int CF_OFF_BAR = CF_OFF_P + CF_P_REGION;
constexpr int CF_NBAR = 2 * CF_SP + 2 * CF_SB + 2 * CF_SA_MAX + 2 * CF_NACC_MAX;
constexpr int CF_OFF_TMEM = CF_OFF_BAR + CF_NBAR * 8;
constexpr int CF_OFF_TAB = (CF_OFF_TMEM + 16 + 15) / 16 * 16;
constexpr int CF_ALLOC = CF_OFF_TAB + CF_TAB_PAIRS * 4 + 1024;
static_assert(CF_ALLOC <= 232448, "shared memory budget");
// two CTAs per SM (CT = 2, 128-wide tiles): each CTA holds 3 B stages, the origin-MMA B block, 2 packed
// P slots (or a 4-stage gather ring), and allocates 256 tensor-memory columns: one 128 x 128
// accumulator [0, 128), three A stages [128, 224), origin scales A [224, 232) / B [232, 240), origin
// A [240, 248), block scales [248, 256)
constexpr int CF2_OFF_OB = 3 * CF_B_STAGE;
constexpr int CF2_OFF_P = CF2_OFF_OB + 128 * 128;
constexpr int CF2_OFF_BAR = CF2_OFF_P + 2 * CF_P_SLOT;
constexpr int CF2_OFF_TMEM = CF2_OFF_BAR + CF_NBAR * 8;
constexpr int CF2_OFF_TAB = (CF2_OFF_TMEM + 16 + 15) / 16 * 16;
constexpr int CF2_ALLOC = CF2_OFF_TAB + CF_TAB_PAIRS * 4 + 1024;
static_assert(2 * (CF2_ALLOC + 1024) <= 233472, "two CTAs per SM: shared memory budget");
// warps: NEPI epilogue warps, then the unpack warps NEPI .. NEPI + NUNP - 1, then producer, waiter, MMA issuer
constexpr int CF_HANDOFF_BAR = 1, CF_EPI_BAR = 2;
constexpr uint32_t CF_SF_COL = 480;                // TMEM columns [480, 512): block scales (every byte 2^1)
constexpr uint32_t CF_ACC0 = 0x4B400000u;          // fp32 1.5 * 2^23: the accumulators' integer origin
// origin MMA (omma): A = 64 ones (e2m1 1.0) per row at TMEM columns [448, 456), B = 1.5 in every
// element of a shared-memory block, scales 2^17 (A) and 2^0 (B): D = 64 * 1.5 * 2^17 = 1.5 * 2^23
// exactly, written with enable-input-d = 0 as a tile's first MMA (instead of 128 KB of tcgen05.st
// resets per 128 x 256 tile, the largest tensor-memory traffic of the short-K tiles)
constexpr uint32_t CF_OA_COL = 448, CF_OSFA_COL = 456, CF_OSFB_COL = 464;

#ifdef DG_TRACE
// CTA 0 event timeline (tools/trace_f4.py): [event][stage or tile index] = clock(), in shared memory
constexpr int CF_TN = 96, CF_TE = 16;
__device__ long long g_cf_tl[CF_TE][CF_TN];
__shared__ uint32_t s_cf_tl[CF_TE][CF_TN];
#define CF_EV(e, i) do { if ((int)(i) < CF_TN) s_cf_tl[e][i] = (uint32_t)clock(); } while (0)
#else
#define CF_EV(e, i) do { } while (0)
#endif

__host__ __device__ constexpr uint32_t cf_idesc(int M, int N) {   // kind::mxf4, e2m1 x e2m1, ue8m0, K-major
    return (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(M >> 4) << 24);
}

DG_DEV void cf_mma_ts_init(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t sfa, uint32_t sfb) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%5], 0;\n\t}" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(sfa), "r"(sfb)
        : "memory");
}

// A operand in tensor memory (TA): the unpacked e2m1 stage is written with tcgen05.st, 8 columns
// (32 bytes = 64 nibbles of every row) per K = 64 step
DG_DEV void cf_mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t sfa, uint32_t sfb) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%5], 1;\n\t}" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(sfa), "r"(sfb)
        : "memory");
}

DG_DEV void cf_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa, uint32_t sfb) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%4], [%5], 1;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(sfa), "r"(sfb)
        : "memory");
}

struct CfDiv {
    uint32_t m, s;
};
inline CfDiv cf_div(uint32_t d) {
    uint32_t s = 0;
    while ((1ull << s) < d) ++s;
    return CfDiv{(uint32_t)((((1ull << s) - d) << 32) / d + 1), s};
}
DG_DEV uint32_t cf_fdiv(uint32_t n, CfDiv f) { return (__umulhi(n, f.m) + n) >> f.s; }

struct CfArgs {
    int64_t np, nq;              // output pixels (rows), output channels (columns)
    int32_t nstages, last_ksteps, ntp, ntq, ntiles;
    int32_t direct;              // 1: 1x1 / stride 1: the NHWC tensor is the im2col matrix (TMA slots)
    int32_t i2c;                 // direct mode of a strided 1x1 conv: the slots come through an im2col-mode
                                 // tensor map (element strides = the conv stride; input pixel (n, s ho, s wo))
    // implicit im2col (direct == 0): x [B][H][W][Cb] packed, Cb = C/4 a power of two >= 16
    const uint8_t *X;
    int32_t H, W, Cb_log2, kw, kw_recip, stride, pad, Ho, Wo, kb;
    const uint8_t *padsrc;       // 16 bytes of the pad code, then 16 zero bytes (beyond K)
    CfDiv fd_wo, fd_ho;
    void *D;
    int64_t ldd;
    int32_t has_rq, early_b;
    int32_t omma;                // 1: the accumulators' origin comes from one MMA per tile (no reset stores)
    // shifted window (GM = 2; direct 3x3 / stride 1 / pad 1, C = 64 or 128): tiles of 128 PADDED
    // pixels q in [0, nqv), nqv = B (H+2)(W+2); the window = the WR padded input pixels q0 - Wp - 1
    // .. in e2m1, K chunk j (32 codes, 16 bytes) of row i at j * lbo + 16 i (no swizzle), so tap
    // (r, s) is the view starting r * Wp + s rows down; fetched packed into wring ring slots of wslot
    // bytes (cp.async), nwin windows of wbytes after them
    int32_t Wp, WR, lbo, wslot, wbytes, nwin;
    int32_t wring;               // packed fetch ring slots (2 or 4): the fill's copies run wring tiles ahead
    int32_t wbres;               // window mode, one column block: all weight stages resident (slot s = stage s)
    int32_t w1x1;                // window mode of a 1x1 stride-1 conv: the window is the pair's own 256 pixel
                                 // rows (no halo, no padding), K = C / 64 MMA k-steps per 128-row block
    int32_t wpair;               // window pair mode (64-wide tiles, resident weights): a work item = 256 padded
                                 // pixels, one window feeds two 128-row blocks into two accumulators
    int64_t nqv;
    CfDiv fd_hpwp, fd_wp;
    // 16-bit SIMD requant (host-verified, f16_params): x = clamp(acc + negA, 0, W), code = (x m + c) >> 14
    uint32_t f16_m, f16_c2, f16_w2, f16_na2;
    int32_t f16_tab, f16_thr0m1, f16_accmax;
};

__device__ __align__(16) uint8_t g_cf_pad[4][32];


// int32 output, or a ragged last column tile with requant (exact 64-bit path): out of line, so that
// the common 16-bit loop stays compact (instruction-cache misses were a top stall of this kernel)
__device__ __noinline__ void cf_epilogue_general(const CfArgs &fa, const RequantArgs &rq, uint32_t trow, int64_t p,
                                                 int64_t q0, int ncols) {
    uint32_t origin[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) origin[j] = CF_ACC0;
#pragma unroll 1
    for (int c = 0; c < ncols / 32; ++c) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(trow + 32 * c, v);
        ptx::tmem_ld_wait();
        if (!fa.omma) ptx::tmem_st_32x32b_x32(trow + 32 * c, origin);
        const int64_t qc = q0 + c * 32;
        if (p >= fa.np || qc >= fa.nq) continue;
        int32_t a[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) a[j] = (int32_t)(v[j] - CF_ACC0);
        if (!fa.has_rq) {
            int32_t *dp = reinterpret_cast<int32_t *>(fa.D) + p * fa.ldd + qc;
            if (qc + 32 <= fa.nq && (reinterpret_cast<uintptr_t>(dp) & 15) == 0) {
#pragma unroll
                for (int j = 0; j < 32; j += 4) *reinterpret_cast<int4 *>(dp + j) = make_int4(a[j], a[j + 1], a[j + 2], a[j + 3]);
            } else {
                for (int j = 0; j < 32; ++j)
                    if (qc + j < fa.nq) dp[j] = a[j];
            }
        } else {
            uint32_t o0 = 0, o1 = 0;
            for (int j = 0; j < 32; ++j)
                if (qc + j < fa.nq) {
                    const uint32_t cd = requant_one(rq, a[j], p, qc + j);
                    if (j < 16) o0 |= cd << (2 * j);
                    else o1 |= cd << (2 * (j - 16));
                }
            store_codes32_ts(reinterpret_cast<uint8_t *>(fa.D) + p * fa.ldd + (qc >> 2), o0, o1,
                             (int)((fa.nq - qc + 3) / 4 < 8 ? (fa.nq - qc + 3) / 4 : 8));
        }
    }
}

// TA: A stages in tensor memory (two accumulators, six 32-column A stages) instead of shared memory
// (three accumulators, four 16 KB SW128 stages written with st.shared)
// NUNP: unpack warps, 4 (one group) or 8 (two groups of 4 owning alternate stages, each with its
// own gather ring: more gathers in flight for the implicit convolutions)
// BNT: output channels per tile, 128 (TA: two accumulators) or 256 (one accumulator: the A operand
// is unpacked once per 256 output channels; the epilogue releases it after two load rounds)
// NEPI: epilogue warps, 4 (one per lane quarter) or 8: two groups, which split each 256-wide tile's
// columns (each group loads its 128 columns and releases them: the single accumulator is free after
// one load round) or own alternate tiles of the 128-wide kernel's two accumulators
// CT: CTAs per SM, 1, or 2 (BNT = 128, TA): two independent pipelines per SM on half the tensor and
// shared memory each (one accumulator, three A stages per CTA)
// GM: how the activations arrive: 0 implicit im2col gather (cp.async ring per unpack group), 1 direct
// (1x1 / stride 1: TMA slots of the NHWC tensor), 2 shifted window (3x3 / stride 1 / pad 1: each
// padded input pixel unpacked once per tile into a shared-memory window, 9 row-shifted views of it
// are the A operands of shared-memory MMAs)
template <bool TA, int NUNP, int GM, int BNT, int NEPI, int CT>
__global__ void __launch_bounds__(32 * (3 + NEPI + NUNP), CT)
lut_conv_f4_kernel(const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_b,
                   const __grid_constant__ CfArgs fa, const __grid_constant__ RequantArgs rq) {
    constexpr bool DIRECT = GM == 1, WINM = GM == 2;
    constexpr bool C2 = CT == 2;
    static_assert(!C2 || (BNT == 128 && TA), "two CTAs per SM: 128-wide tiles, A in tensor memory");
    static_assert(BNT == 256 || BNT == 128 || (BNT == 64 && TA), "tile widths 64 (A in tensor memory), 128, 256");
    static_assert(!WINM || (TA && !C2), "shifted window: one CTA per SM");
    // window mode: the windows and their packed fetch ring after the origin-MMA B block
    constexpr int OFF_W = CF_OFF_A + BNT * 128;
    constexpr int BN_ = BNT, SB_ = (C2 || BNT == 256) ? 3 : CF_SB, B_STAGE_ = BNT * CF_KST / 2;   // (96 / 48 KB of B stages)
    // accumulators: 256-wide 1, 128-wide 2 (two CTAs per SM: 1), 64-wide 4
    // (shifted window, 128 wide: 3, so that window pairs of two accumulators are double-buffered; the
    // window is the shared-memory A operand, the tensor-memory A stages are unused)
    constexpr int CF_NACC = TA ? ((C2 || BNT == 256) ? 1 : (BNT == 64 ? 4 : (WINM ? 3 : 2))) : 3, CF_SA = TA ? (C2 ? 3 : 6) : 4;
    constexpr int RW = BNT < 128 ? BNT : 128;   // columns per epilogue load round
    constexpr uint32_t TA0 = CF_NACC * BN_;   // first tensor-memory A column (TA)
    constexpr uint32_t TCOLS = C2 ? 256 : 512;
    constexpr uint32_t SF_COL = C2 ? 248 : CF_SF_COL, SFB_OFF = C2 ? 4 : 16;
    constexpr uint32_t OA_COL = C2 ? 240 : CF_OA_COL, OSFA_COL = C2 ? 224 : CF_OSFA_COL, OSFB_COL = C2 ? 232 : CF_OSFB_COL;
    static_assert(!TA || (WINM ? TA0 : TA0 + CF_SA * 32) <= (C2 ? OSFA_COL : OA_COL), "tensor memory budget");
    constexpr int SP_ = C2 ? 2 : CF_SP, IG_ = C2 ? 4 : CF_IG;
    constexpr int OFF_OB = C2 ? CF2_OFF_OB : CF_OFF_A, OFF_P = C2 ? CF2_OFF_P : CF_OFF_P;
    constexpr int OFF_BAR = C2 ? CF2_OFF_BAR : CF_OFF_BAR, OFF_TMEM = C2 ? CF2_OFF_TMEM : CF_OFF_TMEM;
    constexpr int OFF_TAB = C2 ? CF2_OFF_TAB : CF_OFF_TAB;
    constexpr int CF_UNP0 = NEPI;
    constexpr bool CSPLIT = NEPI == 8 && BNT == 256;   // the two epilogue groups split every tile's columns
    const int ntiles = fa.ntiles;
    constexpr int CF_PROD = CF_UNP0 + NUNP, CF_WAIT = CF_PROD + 1, CF_MMA = CF_PROD + 2, NG = NUNP / 4;
    constexpr int IGG = IG_ / NG;               // gather ring stages per unpack group
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = ptx::smem_u32(smem);
    const uint32_t bar0 = sbase + OFF_BAR;   // (barrier slots laid out for the largest counts)
    auto full_p = [&](int s) { return bar0 + 8 * s; };
    auto empty_p = [&](int s) { return bar0 + 8 * (CF_SP + s); };
    auto full_b = [&](int s) { return bar0 + 8 * (2 * CF_SP + s); };
    auto empty_b = [&](int s) { return bar0 + 8 * (2 * CF_SP + CF_SB + s); };
    auto full_a = [&](int s) { return bar0 + 8 * (2 * CF_SP + 2 * CF_SB + s); };
    auto empty_a = [&](int s) { return bar0 + 8 * (2 * CF_SP + 2 * CF_SB + CF_SA_MAX + s); };
    auto acc_full = [&](int a) { return bar0 + 8 * (2 * CF_SP + 2 * CF_SB + 2 * CF_SA_MAX + a); };
    auto acc_empty = [&](int a) { return bar0 + 8 * (2 * CF_SP + 2 * CF_SB + 2 * CF_SA_MAX + CF_NACC_MAX + a); };
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + OFF_TMEM);
    uint32_t *tab = reinterpret_cast<uint32_t *>(smem + OFF_TAB);
    volatile uint32_t *f16_bad = reinterpret_cast<volatile uint32_t *>(smem + OFF_TMEM + 8);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) *f16_bad = 0u;

    if (warp == CF_PROD) {
        if (lane == 0) {
            if (DIRECT) ptx::tma_prefetch(&tm_p);
            ptx::tma_prefetch(&tm_b);
            for (int s = 0; s < SP_; ++s) {
                ptx::mbar_init(full_p(s), 1);
                ptx::mbar_init(empty_p(s), 8);   // 4 unpack warps x 2 stages per slot (count 2 for a lone stage)
            }
            for (int s = 0; s < SB_; ++s) {
                ptx::mbar_init(full_b(s), 1);
                ptx::mbar_init(empty_b(s), 1);
            }
            for (int s = 0; s < CF_SA; ++s) {
                ptx::mbar_init(full_a(s), WINM ? NUNP : 4);   // (window: every unpack warp fills it)
                ptx::mbar_init(empty_a(s), 1);
            }
            for (int a = 0; a < CF_NACC; ++a) {
                ptx::mbar_init(acc_full(a), 1);
                ptx::mbar_init(acc_empty(a), CSPLIT ? 8 : 4);
            }
            ptx::fence_mbar_init();
        }
        __syncwarp();
        ptx::tmem_alloc(ptx::smem_u32(tmem_slot), TCOLS);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp < 4) {
        // block scales (every byte 2^1: D = sum (a/2 * 2)(v/2 * 2)) and the accumulators' origin
        const uint32_t lanes = (uint32_t)(warp * 32) << 16;
        uint32_t r[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = 0x80808080u;
        if (C2) ptx::tmem_st_32x32b_x8_splat(tmem + SF_COL + lanes, 0x80808080u);
        else ptx::tmem_st_32x32b_x32(tmem + SF_COL + lanes, r);
        if (fa.omma) {   // origin MMA operands: A ones, scales 2^17 (A) / 2^0 (B); B block of 1.5 in smem
            ptx::tmem_st_32x32b_x8_splat(tmem + OA_COL + lanes, 0x22222222u);
            ptx::tmem_st_32x32b_x8_splat(tmem + OSFA_COL + lanes, 0x90909090u);
            ptx::tmem_st_32x32b_x8_splat(tmem + OSFB_COL + lanes, 0x7F7F7F7Fu);
            if (!C2) ptx::tmem_st_32x32b_x8_splat(tmem + OSFB_COL + 8 + lanes, 0x7F7F7F7Fu);
            for (int i = threadIdx.x; i < BN_ * 128 / 16; i += 128)
                *reinterpret_cast<uint4 *>(smem + OFF_OB + 16 * i) = make_uint4(0x33333333u, 0x33333333u, 0x33333333u, 0x33333333u);
            ptx::fence_proxy_async_smem();
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = CF_ACC0;
#pragma unroll
            for (int c = 0; c < CF_NACC * BN_ / 32; ++c) ptx::tmem_st_32x32b_x32(tmem + (uint32_t)(c * 32) + lanes, r);
        }
        ptx::tmem_st_wait();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x == 0) ptx::griddep_launch_dependents();

    if (warp == CF_PROD) {
        // (weights are read before the programmatic-dependent-launch wait only under early_weights)
        if (!fa.early_b || DIRECT) ptx::griddep_wait();
        uint32_t gp = 0, gb = 0;
        // (pinned in a register: a kernel-parameter load inside the loop slowed the one-slot tiles' producer)
        const uint32_t pi2c = DIRECT ? __shfl_sync(0xffffffffu, (uint32_t)fa.i2c, 0) : 0u;
        if (WINM && fa.wbres) {   // resident weights: every stage loaded once, into slot s (one column block)
            if (lane == 0 && (int)blockIdx.x < ntiles)
                for (int s = 0; s < fa.nstages; ++s) {
                    ptx::mbar_arrive_expect_tx(full_b(s), (uint32_t)B_STAGE_);
                    ptx::tma_load_2d(sbase + CF_OFF_B + s * B_STAGE_, &tm_b, full_b(s), s * (CF_KST / 2), 0);
                }
            __syncwarp();
        } else
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int tq = t % fa.ntq, tp = t / fa.ntq;
            for (int s = 0; s < fa.nstages; ++s, ++gb) {
                if (DIRECT && (s & 1) == 0) {   // a packed slot = 2 stages of every pixel row
                    const int ps = (int)(gp % SP_);
                    ptx::mbar_wait(empty_p(ps), ((gp / SP_) & 1u) ^ 1u);
                    if (lane == 0) {
                        ptx::mbar_arrive_expect_tx(full_p(ps), (uint32_t)CF_P_SLOT);
                        if (pi2c) {   // the tile's first output pixel (n, ho, wo) -> input (n, s ho, s wo)
                            const uint32_t p0 = (uint32_t)tp * CF_BM, tt = cf_fdiv(p0, fa.fd_wo), n = cf_fdiv(tt, fa.fd_ho);
                            ptx::tma_load_im2col_4d(sbase + OFF_P + ps * CF_P_SLOT, &tm_p, full_p(ps), s * (CF_KST / 4),
                                                    (int32_t)(p0 - tt * (uint32_t)fa.Wo) * fa.stride,
                                                    (int32_t)(tt - n * (uint32_t)fa.Ho) * fa.stride, (int32_t)n);
                        } else {
                            ptx::tma_load_2d(sbase + OFF_P + ps * CF_P_SLOT, &tm_p, full_p(ps), s * (CF_KST / 4), tp * CF_BM);
                        }
                    }
                    __syncwarp();
                    ++gp;
                }
                const int bs = (int)(gb % SB_);
                ptx::mbar_wait(empty_b(bs), ((gb / SB_) & 1u) ^ 1u);
                if (lane == 0) {
                    ptx::mbar_arrive_expect_tx(full_b(bs), (uint32_t)B_STAGE_);
                    ptx::tma_load_2d(sbase + CF_OFF_B + bs * B_STAGE_, &tm_b, full_b(bs), s * (CF_KST / 2), tq * BN_);
                    CF_EV(0, gb);
                }
                __syncwarp();
            }
        }
    } else if (warp == CF_WAIT) {
        uint32_t g = 0, tl = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
            if (BNT <= 128 && WINM && fa.wpair) {   // both accumulators of the pair
                ptx::mbar_wait(acc_empty((2 * tl) % CF_NACC), (((2 * tl) / CF_NACC) & 1u) ^ 1u);
                ptx::mbar_wait(acc_empty((2 * tl + 1) % CF_NACC), (((2 * tl + 1) / CF_NACC) & 1u) ^ 1u);
            } else if (CF_NACC > 1) {
                ptx::mbar_wait(acc_empty(tl % CF_NACC), ((tl / CF_NACC) & 1u) ^ 1u);
            }
            if (lane == 0) CF_EV(1, tl);
            if (WINM) ptx::mbar_wait(full_a((int)(tl % (uint32_t)fa.nwin)), (tl / (uint32_t)fa.nwin) & 1u);   // the tile's window
            if (WINM && fa.wbres) {   // resident weights: waited for once; one hand-off per tile
                if (lane == 0) CF_EV(2, tl);
                if (tl == 0)
                    for (int s = 0; s < fa.nstages; ++s) ptx::mbar_wait(full_b(s), 0u);
                ptx::named_bar_sync(CF_HANDOFF_BAR, 64);
                continue;
            }
            for (int s = 0; s < fa.nstages; ++s, ++g) {
                if (!WINM) ptx::mbar_wait(full_a(g % CF_SA), (g / CF_SA) & 1u);
                if (lane == 0) CF_EV(2, g);
                ptx::mbar_wait(full_b(g % SB_), (g / SB_) & 1u);
                if (lane == 0) CF_EV(3, g);
                ptx::named_bar_sync(CF_HANDOFF_BAR, 64);
            }
        }
    } else if (warp == CF_MMA) {
        constexpr uint32_t idesc = cf_idesc(CF_BM, BN_);
        const uint32_t sfa = tmem + SF_COL, sfb = tmem + SF_COL + SFB_OFF;
        const int nst = fa.nstages, lastk = fa.last_ksteps;   // (in registers before any MMA is queued)
        const bool omma = fa.omma != 0;
        // window geometry in registers before any MMA is queued (a parameter load between two
        // tcgen05.mma waits for the queued MMAs): tap (r, s) starts r * Wp + s rows down (16 B each);
        // the second 64-code chunk of a 128-channel tap is 2 K chunks (2 lbo) further
        uint32_t w_tap[9];
#pragma unroll
        for (int q = 0; q < 9; ++q) w_tap[q] = WINM ? (uint32_t)((q / 3) * fa.Wp + q % 3) : 0u;
        const uint32_t w_c2 = WINM ? (uint32_t)(fa.lbo >> 3) : 0u, w_sh = WINM ? (uint32_t)(fa.Cb_log2 - 4) : 0u;
        const uint32_t w_base = sbase + OFF_W + (WINM ? (uint32_t)(fa.wring * fa.wslot) : 0u), w_bytes = WINM ? (uint32_t)fa.wbytes : 0u;
        const uint32_t w_nwin = WINM ? (uint32_t)fa.nwin : 1u, w_lbo = WINM ? (uint32_t)fa.lbo : 0u;
        const bool wbres = WINM && fa.wbres != 0, wpair = WINM && fa.wpair != 0, w1x1 = WINM && fa.w1x1 != 0;
        const int w_nks = WINM ? (1 << fa.Cb_log2) / 16 : 0;   // (1x1: 64-code k-steps per row)
        uint32_t g = 0, tl = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
            const uint32_t acc = tl % CF_NACC;
            const uint32_t dt = tmem + acc * BN_;
            const uint32_t wb = WINM ? tl % w_nwin : 0u;
            const uint64_t aw = WINM ? ptx::desc_k_none(w_base + wb * w_bytes, w_lbo) : 0ull;
            // a single accumulator (256-wide tiles) is waited for here, in parallel with the waiter's
            // stage-0 operand waits (-0.3..0.7 us per layer); with several, the MMA warp must not
            // block (an mbarrier probe here waits behind its queued MMAs: +2 us on the 64 / 128-wide
            // K = 256 layers), the waiter takes it
            if (CF_NACC == 1) ptx::mbar_wait(acc_empty(acc), (tl & 1u) ^ 1u);
            if constexpr (WINM) {
                if (wbres) {   // resident weights (stage s in slot s): the tile's MMAs after one hand-off
                    ptx::named_bar_sync(CF_HANDOFF_BAR, 64);
                    if (lane == 0) CF_EV(14, tl);
                    ptx::tc_fence_after();
                    if (omma && !(BNT <= 128 && wpair))
                        cf_mma_ts_init(dt, tmem + OA_COL, ptx::desc_k_sw128(sbase + OFF_OB), idesc, tmem + OSFA_COL,
                                       tmem + OSFB_COL);
                    // fully unrolled (C = 64: 9 k-steps of 64 codes, one per tap; C = 128: 18, two per
                    // tap): every descriptor is the tile's window / the resident B base plus a constant
                    // (a select chain per MMA paced the warp at ~175 cycles per MMA)
                    const uint64_t bd0 = ptx::desc_k_sw128(sbase + CF_OFF_B);
                    if (BNT <= 128 && wpair) {   // two 128-row blocks of one window: rows [128 h, 128 h + 128)
#pragma unroll 1
                        for (uint32_t h = 0; h < 2; ++h) {
                            const uint32_t va = (2 * tl + h) % CF_NACC, dth = tmem + va * BN_;
                            const uint64_t awh = aw + 128u * h;   // 128 rows x 16 B further down
                            if (omma)
                                cf_mma_ts_init(dth, tmem + OA_COL, ptx::desc_k_sw128(sbase + OFF_OB), idesc,
                                               tmem + OSFA_COL, tmem + OSFB_COL);
                            if (w1x1) {   // 1x1: k-step j = 64-code chunk j of the pixel's own row
#pragma unroll
                                for (int j = 0; j < 4; ++j) {
                                    if (j >= w_nks) break;
                                    cf_mma(dth, awh + (uint64_t)(j * w_c2), bd0 + 2 * j, idesc, sfa, sfb);
                                }
                            } else if (w_sh == 0) {
#pragma unroll
                                for (int j = 0; j < 9; ++j)
                                    cf_mma(dth, awh + (uint64_t)w_tap[j],
                                           bd0 + (uint64_t)(((j >> 2) * B_STAGE_) >> 4) + 2 * (j & 3), idesc, sfa, sfb);
                            } else {
#pragma unroll
                                for (int j = 0; j < 18; ++j)
                                    cf_mma(dth, awh + (uint64_t)(w_tap[j >> 1] + (j & 1) * w_c2),
                                           bd0 + (uint64_t)(((j >> 2) * B_STAGE_) >> 4) + 2 * (j & 3), idesc, sfa, sfb);
                            }
                            ptx::mma_commit_warp(acc_full((int)va));
                        }
                        if (lane == 0) CF_EV(15, tl);
                        ptx::mma_commit_warp(empty_a((int)wb));   // the window is free again
                        __syncwarp();
                        continue;
                    }
                    if (w_sh == 0) {
#pragma unroll
                        for (int j = 0; j < 9; ++j)
                            cf_mma(dt, aw + (uint64_t)w_tap[j], bd0 + (uint64_t)(((j >> 2) * B_STAGE_) >> 4) + 2 * (j & 3),
                                   idesc, sfa, sfb);
                    } else {
#pragma unroll
                        for (int j = 0; j < 18; ++j)
                            cf_mma(dt, aw + (uint64_t)(w_tap[j >> 1] + (j & 1) * w_c2),
                                   bd0 + (uint64_t)(((j >> 2) * B_STAGE_) >> 4) + 2 * (j & 3), idesc, sfa, sfb);
                    }
                    if (lane == 0) CF_EV(15, tl);
                    ptx::mma_commit_warp(empty_a((int)wb));   // the window is free again
                    ptx::mma_commit_warp(acc_full(acc));
                    __syncwarp();
                    continue;
                }
            }
            for (int s = 0; s < nst; ++s, ++g) {
                const int sa = (int)(g % CF_SA), bs = (int)(g % SB_);
                ptx::named_bar_sync(CF_HANDOFF_BAR, 64);
                if (lane == 0) CF_EV(14, g);
                ptx::tc_fence_after();
                if (TA && omma && s == 0)
                    cf_mma_ts_init(dt, tmem + OA_COL, ptx::desc_k_sw128(sbase + OFF_OB), idesc, tmem + OSFA_COL,
                                   tmem + OSFB_COL);
                const uint64_t ad = ptx::desc_k_sw128(sbase + CF_OFF_A + sa * CF_A_STAGE);
                const uint64_t bd = ptx::desc_k_sw128(sbase + CF_OFF_B + bs * B_STAGE_);
                const uint32_t at = tmem + TA0 + (uint32_t)(sa * 32);
                if constexpr (WINM) {   // k-step j = 4 s + k: tap j >> w_sh, 64-code chunk j & w_sh of it
                    const int nk = s < nst - 1 ? 4 : lastk;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (k >= nk) break;
                        const uint32_t j = (uint32_t)(4 * s + k), tap = j >> w_sh;
                        uint32_t toff = w_tap[0];
#pragma unroll
                        for (int q = 1; q < 9; ++q) toff = tap == (uint32_t)q ? w_tap[q] : toff;
                        cf_mma(dt, aw + (uint64_t)(toff + (j & w_sh) * w_c2), bd + 2 * k, idesc, sfa, sfb);
                    }
                    if (lane == 0) CF_EV(15, g);
                    ptx::mma_commit_warp(empty_b(bs));
                    if (s == nst - 1) {
                        ptx::mma_commit_warp(empty_a((int)wb));   // the window is free again
                        ptx::mma_commit_warp(acc_full(acc));
                    }
                    __syncwarp();
                    continue;
                }
                if (s < nst - 1) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if constexpr (TA) cf_mma_ts(dt, at + 8 * k, bd + 2 * k, idesc, sfa, sfb);
                        else cf_mma(dt, ad + 2 * k, bd + 2 * k, idesc, sfa, sfb);
                    }
                } else {
                    for (int k = 0; k < lastk; ++k) {
                        if constexpr (TA) cf_mma_ts(dt, at + 8 * k, bd + 2 * k, idesc, sfa, sfb);
                        else cf_mma(dt, ad + 2 * k, bd + 2 * k, idesc, sfa, sfb);
                    }
                }
                if (lane == 0) CF_EV(15, g);
                ptx::mma_commit_warp(empty_a(sa));
                ptx::mma_commit_warp(empty_b(bs));
                if (s == nst - 1) ptx::mma_commit_warp(acc_full(acc));
                __syncwarp();
                if (lane == 0) CF_EV(4, g);
            }
        }
    } else if (WINM && warp >= CF_UNP0 && fa.w1x1) {
        // ---------------- 1x1 window fill: thread = one of the pair's 256 pixel rows; its packed pixel
        // (C/4 bytes, up to 64) arrives by cp.async two pairs ahead, becomes e2m1 nibbles chunk by
        // chunk (16 packed bytes -> two 16-byte K chunks at j * lbo + 16 * row)
        ptx::griddep_wait();
        const int tid = (warp - CF_UNP0) * 32 + lane;
        const int cb = 1 << fa.Cb_log2, nch = cb >> 4;
        const uint32_t ring = sbase + OFF_W, wins = ring + 2u * (uint32_t)fa.wslot;
        auto fetch = [&](int t, int slot) {
            if (t < ntiles && tid < fa.WR) {
                const int64_t q = (int64_t)(t / fa.ntq) * (2 * CF_BM) + tid;
                const uint8_t *src = q < fa.nqv ? fa.X + (q << fa.Cb_log2) : fa.padsrc;
                const uint32_t dst = ring + (uint32_t)(slot * fa.wslot + tid * cb);
                for (int c = 0; c < nch; ++c) ptx::cp_async16(dst + 16 * c, q < fa.nqv ? src + 16 * c : fa.padsrc);
            }
            ptx::cp_async_commit();
        };
        fetch(blockIdx.x, 0);
        fetch(blockIdx.x + gridDim.x, 1);
        uint32_t tl = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
            const int slot = (int)(tl & 1u), wb = (int)(tl % (uint32_t)fa.nwin);
            ptx::cp_async_wait<1>();
            ptx::mbar_wait(empty_a(wb), ((tl / (uint32_t)fa.nwin) & 1u) ^ 1u);   // the window's previous pair finished
            if (tid < fa.WR) {
                const uint32_t wdst = wins + (uint32_t)(wb * fa.wbytes + tid * 16);
                for (int c = 0; c < nch; ++c) {
                    const uint4 v = ptx::lds128(ring + (uint32_t)(slot * fa.wslot + tid * cb + 16 * c));
                    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
                    uint32_t e[8];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        e[2 * k] = w[k] & 0x33333333u;
                        e[2 * k + 1] = (w[k] >> 2) & 0x33333333u;
                    }
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(wdst + (uint32_t)(2 * c * fa.lbo)),
                                 "r"(e[0]), "r"(e[1]), "r"(e[2]), "r"(e[3]) : "memory");
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(wdst + (uint32_t)((2 * c + 1) * fa.lbo)),
                                 "r"(e[4]), "r"(e[5]), "r"(e[6]), "r"(e[7]) : "memory");
                }
            }
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(full_a(wb));
            fetch(t + 2 * (int)gridDim.x, slot);   // (after the fence: see the 3x3 fill)
        }
    } else if (WINM && warp >= CF_UNP0) {
        // ---------------- window fill: thread = window row(s) (padded input pixels q0 - Wp - 1 + row):
        // the packed pixel (C/4 bytes) arrives by cp.async two tiles ahead (ring of 2 slots), becomes
        // e2m1 nibbles (the two masks per 16 codes) and is stored as C/32 16-byte K chunks (chunk j
        // at j * lbo + 16 * row); all NUNP warps fill each tile's window
        ptx::griddep_wait();
        constexpr int NT = NUNP * 32, WMAXR = 3;
        const int tid = (warp - CF_UNP0) * 32 + lane;
        const int cb = 1 << fa.Cb_log2, nch = cb >> 4;   // packed bytes per pixel (16 / 32), 16-byte chunks
        const int nrt = (fa.WR + NT - 1) / NT;            // window rows per thread (host: <= 3)
        const uint32_t ring = sbase + OFF_W, wins = ring + (uint32_t)(fa.wring * fa.wslot);
        const int wring = fa.wring;
        auto fetch = [&](int t, int slot) {
            if (t < ntiles) {
                const int tp = t / fa.ntq;
                for (int i = 0; i < nrt; ++i) {
                    const int row = tid + i * NT;
                    if (row >= fa.WR) break;
                    const int64_t q = (int64_t)tp * (fa.wpair ? 2 * CF_BM : CF_BM) - (fa.Wp + 1) + row;   // padded pixel of this row
                    const uint8_t *src = nullptr;
                    if (q >= 0 && q < fa.nqv) {
                        const uint32_t b = cf_fdiv((uint32_t)q, fa.fd_hpwp);
                        const uint32_t rem = (uint32_t)q - b * (uint32_t)((fa.H + 2) * fa.Wp);
                        const uint32_t hp = cf_fdiv(rem, fa.fd_wp), wp = rem - hp * (uint32_t)fa.Wp;
                        if (hp >= 1 && hp <= (uint32_t)fa.H && wp >= 1 && wp <= (uint32_t)fa.W)
                            src = fa.X + ((((int64_t)b * fa.H + hp - 1) * fa.W + wp - 1) << fa.Cb_log2);
                    }
                    const uint32_t dst = ring + (uint32_t)(slot * fa.wslot + row * cb);
                    for (int c = 0; c < nch; ++c) ptx::cp_async16(dst + 16 * c, src ? src + 16 * c : fa.padsrc);
                }
            }
            ptx::cp_async_commit();
        };
        for (int i = 0; i < wring; ++i) fetch(blockIdx.x + i * (int)gridDim.x, i);
        uint32_t tl = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
            const int slot = (int)(tl % (uint32_t)wring), wb = (int)(tl % (uint32_t)fa.nwin);
            // this tile's copies (the oldest group; each thread reads its own rows)
            if (wring == 4) ptx::cp_async_wait<3>();
            else ptx::cp_async_wait<1>();
            if (threadIdx.x == (CF_UNP0 + NUNP - 1) * 32) CF_EV(12, tl);
            uint32_t e[WMAXR][16];
#pragma unroll
            for (int i = 0; i < WMAXR; ++i) {
                const int row = tid + i * NT;
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const uint4 v = (i < nrt && row < fa.WR && c < nch) ? ptx::lds128(ring + (uint32_t)(slot * fa.wslot + row * cb + 16 * c))
                                                                        : make_uint4(0, 0, 0, 0);
                    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        e[i][8 * c + 2 * k] = w[k] & 0x33333333u;
                        e[i][8 * c + 2 * k + 1] = (w[k] >> 2) & 0x33333333u;
                    }
                }
            }
            ptx::mbar_wait(empty_a(wb), ((tl / (uint32_t)fa.nwin) & 1u) ^ 1u);   // the window's previous tile finished
            if (threadIdx.x == CF_UNP0 * 32) CF_EV(13, tl);
#pragma unroll
            for (int i = 0; i < WMAXR; ++i) {
                const int row = tid + i * NT;
                if (i >= nrt || row >= fa.WR) break;
                const uint32_t wdst = wins + (uint32_t)(wb * fa.wbytes + row * 16);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (j >= 2 * nch) break;
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(wdst + (uint32_t)(j * fa.lbo)),
                                 "r"(e[i][4 * j]), "r"(e[i][4 * j + 1]), "r"(e[i][4 * j + 2]), "r"(e[i][4 * j + 3])
                                 : "memory");
                }
            }
            ptx::fence_proxy_async_smem();   // generic-proxy stores -> visible to the tensor core
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(full_a(wb));
            if (threadIdx.x == CF_UNP0 * 32) CF_EV(5, tl);
            if (threadIdx.x == (CF_UNP0 + NUNP - 1) * 32) CF_EV(0, tl);
            // the slot's bytes are in registers: refill it, after the window's proxy fence (a fence
            // behind freshly issued cp.async copies waited for them to land: ~1000 cycles per tile)
            fetch(t + wring * (int)gridDim.x, slot);
        }
    } else if (warp >= CF_UNP0) {
        // thread = pixel row r of the tile: 64 packed bytes (256 codes) per stage -> 32 words of e2m1
        // nibbles (x & 0x33333333, (x >> 2) & 0x33333333 per packed word) -> A stage.  Group grp owns
        // the stages g with g % NG == grp.
        ptx::griddep_wait();
        const int grp = (warp - CF_UNP0) >> 2;
        const int r = (warp & 3) * 32 + lane;
        uint32_t g = 0, gp = 0, own = 0;
        // implicit gather cursor of this group: work item gt, stage gs of the next fetch; this row's pixel
        int gt = blockIdx.x, gs = grp;
        const uint8_t *img = fa.X;
        int32_t h0 = 0, w0 = 0;
        auto pixel = [&]() {
            const int64_t p = (int64_t)(gt / fa.ntq) * CF_BM + r;
            const uint32_t pp = (uint32_t)(p < fa.np ? p : fa.np - 1);
            const uint32_t tt = cf_fdiv(pp, fa.fd_wo), b = cf_fdiv(tt, fa.fd_ho);
            img = fa.X + (((int64_t)b * fa.H * fa.W) << fa.Cb_log2);
            h0 = (int32_t)(tt - b * (uint32_t)fa.Ho) * fa.stride - fa.pad;
            w0 = (int32_t)(pp - tt * (uint32_t)fa.Wo) * fa.stride - fa.pad;
        };
        auto settle = [&]() {   // move (gt, gs) into the work item that holds stage gs
            bool moved = false;
            while (gs >= fa.nstages && gt < ntiles) { gs -= fa.nstages; gt += gridDim.x; moved = true; }
            if (moved && gt < ntiles) pixel();
        };
        const uint32_t ring = sbase + OFF_P + (uint32_t)(grp * IGG * CF_RING) + (uint32_t)(r * 64);
        auto fetch = [&](int slot) {   // the cursor's stage -> ring slot; advance the cursor by NG stages
            if (gt < ntiles) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int32_t byte = gs * 64 + 16 * c;
                    const int32_t tap = byte >> fa.Cb_log2, off = byte & ((1 << fa.Cb_log2) - 1);
                    const int32_t rr = (tap * fa.kw_recip) >> 16, ss = tap - rr * fa.kw;
                    const int32_t hi = h0 + rr, wi = w0 + ss;
                    const uint8_t *src = byte >= fa.kb ? fa.padsrc + 16
                                         : ((uint32_t)hi < (uint32_t)fa.H && (uint32_t)wi < (uint32_t)fa.W)
                                               ? img + ((((int64_t)hi * fa.W + wi) << fa.Cb_log2) + off)
                                               : fa.padsrc;
                    ptx::cp_async16(ring + (uint32_t)(slot * CF_RING) + ((c ^ ((r >> 1) & 3)) << 4), src);
                }
                gs += NG;
                settle();
            }
            ptx::cp_async_commit();
        };
        if (!DIRECT) {
            if (gt < ntiles) pixel();
            settle();
            for (int i = 0; i < IGG; ++i) fetch(i);
        }
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            for (int s = 0; s < fa.nstages; ++s, ++g) {
                const bool slot_end = (s & 1) == 1 || s == fa.nstages - 1;   // last stage of a packed slot
                if (NG > 1 && (int)(g % NG) != grp) {   // another group's stage: slot bookkeeping only
                    if (DIRECT && slot_end) ++gp;
                    continue;
                }
                uint4 v[4];
                if (DIRECT) {
                    const int ps = (int)(gp % SP_), sub = s & 1;
                    ptx::mbar_wait(full_p(ps), (gp / SP_) & 1u);
                    if (threadIdx.x == CF_UNP0 * 32) CF_EV(12, g);
                    const uint32_t pbase = sbase + OFF_P + ps * CF_P_SLOT;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {   // SW128 slot: 16-byte unit XOR row bits
                        const uint32_t lin = (uint32_t)(r * 128 + sub * 64 + 16 * c);
                        v[c] = ptx::lds128(pbase + (lin ^ (((lin >> 7) & 7u) << 4)));
                    }
                    // this stage's share of the slot is released once its loads have landed
                    // (release_after_loads: the refilling TMA raced with outstanding loads, measured
                    // nondeterministic rows); a slot's lone last stage counts twice
                    ptx::release_after_loads(empty_p(ps), (s & 1) == 0 && s == fa.nstages - 1 ? 2u : 1u,
                                             v[0].x ^ v[1].x ^ v[2].x ^ v[3].x);
                    if (slot_end) ++gp;
                } else {
                    ptx::cp_async_wait<IGG - 1>();   // this stage's copies (the oldest group) landed
                    if ((warp & 3) == 0 && lane == 0) CF_EV(12, g);
                    const int slot = (int)(own % IGG);
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        v[c] = ptx::lds128(ring + (uint32_t)(slot * CF_RING) + ((c ^ ((r >> 1) & 3)) << 4));
                    fetch(slot);   // values are in registers: refill the slot IGG own stages ahead
                }
                ++own;
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
                const int sa = (int)(g % CF_SA);
                ptx::mbar_wait(empty_a(sa), ((g / CF_SA) & 1u) ^ 1u);
                if ((warp & 3) == 0 && lane == 0) CF_EV(13, g);
                if constexpr (TA) {   // row r = lane quarter (warp & 3) x 32 + lane: 32 columns of this stage
                    ptx::tc_fence_after();
                    ptx::tmem_st_32x32b_x32(tmem + TA0 + (uint32_t)(sa * 32) + ((uint32_t)((warp & 3) * 32) << 16), e);
                    ptx::tmem_st_wait();
                    ptx::tc_fence_before();
                } else {
                    // SW128 K-major A stage: row r at (r/8)*1024 + (r%8)*128, 16-byte chunk j at (j ^ (r%8))*16
                    const uint32_t row = sbase + CF_OFF_A + sa * CF_A_STAGE + (uint32_t)((r >> 3) * 1024 + (r & 7) * 128);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(row + (uint32_t)(((j ^ (r & 7)) << 4))),
                                     "r"(e[4 * j]), "r"(e[4 * j + 1]), "r"(e[4 * j + 2]), "r"(e[4 * j + 3])
                                     : "memory");
                    ptx::fence_proxy_async_smem();
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(full_a(sa));
                if ((warp & 3) == 0 && lane == 0) CF_EV(5, g);
            }
        }
    } else {
        // ---------------- epilogue (lane quarter = warp)
        const int quarter = warp & 3, eg = warp >> 2;
        if (!fa.early_b) ptx::griddep_wait();   // (the bias may come from the previous kernel)
        if (fa.has_rq && fa.f16_tab) {   // per-column 16-bit offsets: negA = bias - (thr0 - 1)
            uint32_t bad = 0;
            for (int i = threadIdx.x; i < (int)(fa.nq >> 1); i += NEPI * 32) {
                const int64_t n0 = (int64_t)__ldg(rq.bias + 2 * i) - fa.f16_thr0m1;
                const int64_t n1 = (int64_t)__ldg(rq.bias + 2 * i + 1) - fa.f16_thr0m1;
                if ((n0 < 0 ? -n0 : n0) + fa.f16_accmax > 32767 || (n1 < 0 ? -n1 : n1) + fa.f16_accmax > 32767) bad = 1;
                tab[i] = ((uint32_t)n0 & 0xFFFFu) | ((uint32_t)n1 << 16);
            }
            if (bad) *f16_bad = 1u;   // some offset overflows int16: every tile takes the exact path
            ptx::named_bar_sync(CF_EPI_BAR, NEPI * 32);
        }
        const bool f16_ok = fa.has_rq && *f16_bad == 0u;
        ptx::griddep_wait();
        const uint32_t tabs = sbase + OFF_TAB;
        uint32_t tl = 0;
        constexpr int RD_N = CSPLIT ? 1 : BN_ / RW;   // load rounds per warp and tile
        const bool epair = BNT <= 128 && WINM && fa.wpair != 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl)
        for (int h = 0; h < (epair ? 2 : 1); ++h) {
            // v: the accumulator sequence number (pair mode: two 128-row blocks per work item)
            const uint32_t v = epair ? 2 * tl + (uint32_t)h : tl;
            if (NEPI == 8 && !CSPLIT && (int)(v & 1u) != eg) continue;   // the other group's accumulator
            const int tq = t % fa.ntq, tp = epair ? 2 * (t / fa.ntq) + h : t / fa.ntq;
            int64_t p = (int64_t)tp * CF_BM + quarter * 32 + lane;
            if (WINM && !fa.w1x1) {   // padded pixel -> output pixel row, or np (not stored) for a padding position
                const int64_t q = p;
                p = fa.np;
                if (q < fa.nqv) {
                    const uint32_t b = cf_fdiv((uint32_t)q, fa.fd_hpwp);
                    const uint32_t rem = (uint32_t)q - b * (uint32_t)((fa.H + 2) * fa.Wp);
                    const uint32_t hp = cf_fdiv(rem, fa.fd_wp), wp = rem - hp * (uint32_t)fa.Wp;
                    if (hp >= 1 && hp <= (uint32_t)fa.H && wp >= 1 && wp <= (uint32_t)fa.W)
                        p = ((int64_t)b * fa.H + hp - 1) * fa.W + wp - 1;
                }
            }
            const int64_t q0 = (int64_t)tq * BN_;
            const uint32_t acc = v % CF_NACC;
            ptx::mbar_wait(acc_full(acc), (v / CF_NACC) & 1u);
            if (lane == 0 && quarter == 0) CF_EV(6 + 3 * eg, v);
            ptx::tc_fence_after();
            const int c0 = CSPLIT ? eg * 128 : 0;   // this warp's first column of the tile
            const uint32_t trow = tmem + acc * BN_ + (uint32_t)c0 + ((uint32_t)(quarter * 32) << 16);
            if (f16_ok && q0 + BN_ <= fa.nq) {
#pragma unroll 1
              for (int rd = 0; rd < RD_N; ++rd) {   // RW columns per load round
                const uint32_t trd = trow + (uint32_t)(rd * RW);
                const int64_t q0r = q0 + c0 + rd * RW;
                uint32_t r16[RW / 64][32];   // the round's columns as 16-bit pairs (low halves = the integer values)
#pragma unroll
                for (int l = 0; l < RW / 64; ++l) ptx::tmem_ld_32x32b_x32_pack16(trd + 64 * l, r16[l]);
                ptx::tmem_ld_wait();
                if (!fa.omma) {
#pragma unroll
                    for (int c = 0; c < RW / 8; ++c) ptx::tmem_st_32x32b_x8_splat(trd + 8 * c, CF_ACC0);   // reset to the origin
                    ptx::tmem_st_wait();
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0 && rd == RD_N - 1) ptx::mbar_arrive(acc_empty(acc));
                if (lane == 0 && quarter == 0) CF_EV(7 + 3 * eg, v);
                if (p < fa.np) {
#pragma unroll
                    for (int hh = 0; hh < RW / 32; ++hh) {
                        const int64_t qc = q0r + hh * 32;
                        uint32_t na[16];
                        if (fa.f16_tab) {
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const uint4 t4 = ptx::lds128(tabs + (uint32_t)(qc >> 1) * 4u + 16 * j);
                                na[4 * j] = t4.x; na[4 * j + 1] = t4.y; na[4 * j + 2] = t4.z; na[4 * j + 3] = t4.w;
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < 16; ++j) na[j] = fa.f16_na2;
                        }
                        uint32_t rr[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) rr[j] = r16[hh >> 1][16 * (hh & 1) + j];
                        const uint2 o = requant16_32(rr, na, fa.f16_w2, fa.f16_m, fa.f16_c2);
                        uint8_t *dp = reinterpret_cast<uint8_t *>(fa.D) + p * fa.ldd + (qc >> 2);
                        if ((reinterpret_cast<uintptr_t>(dp) & 7) == 0) *reinterpret_cast<uint2 *>(dp) = o;
                        else store_codes32_ts(dp, o.x, o.y, 8);
                    }
                }
              }
            } else {   // int32 output, or the ragged last column tile with requant (exact 64-bit path)
                cf_epilogue_general(fa, rq, trow, p, q0 + c0, CSPLIT ? 128 : BN_);
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(acc_empty(acc));
            }
            if (lane == 0 && quarter == 0) CF_EV(8 + 3 * eg, v);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
#ifdef DG_TRACE
    if (blockIdx.x == 0)
        for (int i = threadIdx.x; i < CF_TE * CF_TN; i += blockDim.x) (&g_cf_tl[0][0])[i] = (&s_cf_tl[0][0])[i];
#endif
    if (warp == CF_PROD) ptx::tmem_dealloc(tmem, TCOLS);
}

typedef CUresult (*CfEncode)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool cf_map(CUtensorMap *m, const void *base, int64_t row_bytes, int64_t ld, int64_t rows, int box_rows) {
    static CfEncode fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<CfEncode>(p);
    }
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)row_bytes, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld};
    cuuint32_t box[2] = {128, (cuuint32_t)box_rows}, estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

const uint8_t *cf_pad_source(int pad_code) {
    static const uint8_t *base = nullptr;
    if (!base) {
        uint8_t h[4][32] = {};
        for (int c = 0; c < 4; ++c)
            for (int i = 0; i < 16; ++i) h[c][i] = (uint8_t)(c | (c << 2) | (c << 4) | (c << 6));
        if (cudaMemcpyToSymbol(g_cf_pad, h, sizeof(h)) != cudaSuccess) return nullptr;
        void *p = nullptr;
        if (cudaGetSymbolAddress(&p, g_cf_pad) != cudaSuccess) return nullptr;
        base = reinterpret_cast<const uint8_t *>(p);
    }
    return base + 32 * (pad_code & 3);
}

}  // namespace

#ifdef DG_TRACE
extern "C" __attribute__((visibility("default"))) int dg_debug_cf_timeline(long long *host, int reset) {
    if (reset) {
        static long long z[CF_TE * CF_TN];
        return cudaMemcpyToSymbol(g_cf_tl, z, sizeof(z)) == cudaSuccess ? 0 : -1;
    }
    return cudaMemcpyFromSymbol(host, g_cf_tl, sizeof(long long) * CF_TE * CF_TN) == cudaSuccess ? 0 : -1;
}
#endif

// Conv (or a 1x1 conv = GEMM in the conv orientation) on the FP4 path.  x: NHWC packed [B][H][W][C/4];
// w4: e2m1 weights [Cout][ld4] (dg_expand_operand_f4 of the packed weights, K order (r, s, c));
// out: int32 [pixels][Cout] or, with rq, packed codes [pixels][Cout/4].  Returns DG_ERR_UNSUPPORTED
// for what this kernel does not cover (the caller then runs the int8 tensor-core path):
// residuals, bias per row, requant parameters without a 16-bit form, channel counts whose taps are
// not 16-byte power-of-two chunks.
typedef CUresult (*CfEncodeIm2col)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const int *, const int *, cuuint32_t, cuuint32_t,
                                   const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// im2col-mode map of a strided 1x1 conv's NHWC input (C = cb bytes per pixel): 128 output pixels x
// 128 channel bytes per load in the direct slots' 128-byte-swizzled row layout
bool cf_map_im2col(CUtensorMap *m, const void *base, int64_t cb, int64_t W, int64_t H, int64_t N, int stride) {
    static CfEncodeIm2col fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<CfEncodeIm2col>(p);
    }
    if (!fn) return false;
    cuuint64_t dims[4] = {(cuuint64_t)cb, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    cuuint64_t strides[3] = {(cuuint64_t)cb, (cuuint64_t)(W * cb), (cuuint64_t)(H * W * cb)};
    int lo[2] = {0, 0}, hi[2] = {0, 0};   // 1x1, no padding: the bounding box is the image
    cuuint32_t es[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void *>(base), dims, strides, lo, hi, 128, CF_BM, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

dg_status lut_conv_f4(const uint8_t *x, const uint8_t *w4, int64_t ld4, const TsConv &cv, int64_t rows, int64_t cout,
                      int64_t K, int64_t acc_bound, void *out, int64_t ldd, const RequantArgs *rq, cudaStream_t st,
                      bool b_prepared) {
    if (rq && (rq->res || rq->res_codes || (rq->bias && rq->bias_axis != 0) || rq->dir <= 0)) return DG_ERR_UNSUPPORTED;
    if (cout > 2 * CF_TAB_PAIRS || rows >= ((int64_t)1 << 31)) return DG_ERR_UNSUPPORTED;
    const int32_t cb = cv.Cb;
    // strided 1x1 convs (downsample) on the direct path through an im2col-mode tensor map (option f4_i2c)
    const bool i2c = cv.kh == 1 && cv.kw == 1 && cv.pad == 0 && cv.stride > 1 && cb % 16 == 0 && opt(OPT_F4_I2C) > 0 &&
                     cv.H < 65536 && cv.W < 65536 && ((uintptr_t)x & 15) == 0;
    bool direct = cv.kh == 1 && cv.kw == 1 && cv.pad == 0 && (cv.stride == 1 || i2c);
    if (!direct && !(cb >= 16 && (cb & (cb - 1)) == 0 && cv.kh * cv.kw <= 64)) return DG_ERR_UNSUPPORTED;
    if (direct && (cb % 16 || ((uintptr_t)x & 15))) return DG_ERR_UNSUPPORTED;
    CfArgs fa{};
    fa.np = rows;
    fa.nq = cout;
    fa.nstages = (int32_t)((K + CF_KST - 1) / CF_KST);
    fa.last_ksteps = (int32_t)(((K - (int64_t)(fa.nstages - 1) * CF_KST) + 63) / 64);
    fa.ntp = (int32_t)((rows + CF_BM - 1) / CF_BM);
    // tile width: 256 output channels (one accumulator, half the gather + unpack work per output) when
    // they divide Cout (a ragged last tile takes the slow exact epilogue), else 128 (option f4_bn: 0
    // auto, 128, 256).  Measured per layer: the 3x3 convs over 256 channels
    // 28.5 -> 18.5 us against 26.3 us at 128 wide.
    const int fbn = (int)opt(OPT_F4_BN);
    const int bnt = fbn == 64 ? 64 : fbn == 128 ? 128 : (fbn == 256 ? 256 : (cout % 256 == 0 ? 256 : (cout <= 64 ? 64 : 128)));
    fa.ntq = (int32_t)((cout + bnt - 1) / bnt);
    // shifted window (option f4_win: 2 (default) for the direct 3x3 / stride 1 / pad 1 convs over 64 or
    // 128 channels whose weights can stay resident (one column block, all stages in the B ring), 1 for
    // every such conv, 0 never): tiles over the padded pixel space, one window per tile (or pair)
    const int64_t fwin = opt(OPT_F4_WIN);
    const bool res_ok = fa.ntq == 1 && fa.nstages <= (bnt == 256 ? 3 : CF_SB) && opt(OPT_F4_WBRES) > 0;
    const bool win3 = !direct && (fwin == 1 || (fwin == 2 && res_ok)) && cv.kh == 3 && cv.kw == 3 && cv.stride == 1 &&
                      cv.pad == 1 && (cb == 16 || cb == 32) && cv.Ho == cv.H && cv.Wo == cv.W;
    // 1x1 stride-1 convs into 64 / 128 channels as window pairs (option f4_w1x1: 1 (default) over 64
    // input channels, 2 over 64 / 128 / 256): the direct path's per-128-row hand-off chain bounds these
    // narrow tiles; a pair's 256 pixel rows are the window.  Measured (ResNet-50 b256): 64 -> 64
    // 24.6 -> 23.1 us; over 256 channels slower (the fill's 4 chunks per row: 25.8 -> 32.3 us)
    const int64_t fw1 = opt(OPT_F4_W1X1);
    const bool w1x1 = direct && !i2c && res_ok && bnt <= 128 && (cb == 16 || (fw1 == 2 && (cb == 32 || cb == 64))) &&
                      fw1 > 0 && opt(OPT_F4_WPAIR) > 0 && fwin != 0;
    const bool win = win3 || w1x1;
    if (w1x1) direct = false;
    if (w1x1) {   // the pixel rows themselves: no halo, no padding, always pairs
        fa.w1x1 = 1;
        fa.Wp = 0;
        fa.nqv = rows;
        fa.wbres = 1;
        fa.wpair = 1;
        fa.ntp = (int32_t)((rows + 2 * CF_BM - 1) / (2 * CF_BM));
        fa.WR = 2 * CF_BM;
        fa.lbo = fa.WR * 16;
        fa.wslot = (fa.WR * cb + 127) / 128 * 128;
        fa.wbytes = (cb / 8) * fa.lbo;
        const int region = CF_OFF_BAR - (CF_OFF_A + bnt * 128);
        fa.wring = 2;
        fa.nwin = (region - 2 * fa.wslot) / fa.wbytes;
        if (fa.nwin > 3) fa.nwin = 3;
        if (fa.nwin < 1) return DG_ERR_UNSUPPORTED;
    } else if (win) {
        const int64_t Wp = cv.W + 2, Hp = cv.H + 2, B = rows / ((int64_t)cv.H * cv.W);
        fa.Wp = (int32_t)Wp;
        fa.nqv = B * Hp * Wp;
        if (fa.nqv >= ((int64_t)1 << 31)) return DG_ERR_SHAPE;
        // one column block whose weight stages all fit the B ring: loaded once, one hand-off per tile
        // (option f4_wbres); with 64 / 128-wide tiles, pair mode (option f4_wpair): one window of 256 + halo
        // rows feeds two 128-row blocks (the halo unpacked once per 256 rows, one hand-off per pair)
        fa.wbres = res_ok ? 1 : 0;
        fa.wpair = (fa.wbres && bnt <= 128 && opt(OPT_F4_WPAIR) > 0 && 2 * CF_BM + 2 * Wp + 2 <= 3 * 8 * 32) ? 1 : 0;
        const int64_t wrows = fa.wpair ? 2 * CF_BM : CF_BM;
        fa.ntp = (int32_t)((fa.nqv + wrows - 1) / wrows);
        fa.WR = (int32_t)((wrows + 2 * Wp + 2 + 7) / 8 * 8);   // multiple of 8 rows: lbo a multiple of 128 B
        if (fa.WR > 3 * 8 * 32) return DG_ERR_UNSUPPORTED;      // (at most 3 window rows per fill thread)
        fa.lbo = fa.WR * 16;
        fa.wslot = (fa.WR * cb + 127) / 128 * 128;
        fa.wbytes = (cb / 8) * fa.lbo;                           // 2 Cb e2m1 bytes per row = Cb / 8 K chunks
        const int region = CF_OFF_BAR - (CF_OFF_A + bnt * 128);
        // fetch ring: 4 slots (copies 4 tiles ahead: their latency under load exceeded two tiles) when
        // that leaves room for a window, else 2
        fa.wring = (region - 4 * fa.wslot) / fa.wbytes >= 2 ? 4 : 2;   // (two windows at least)
        fa.nwin = (region - fa.wring * fa.wslot) / fa.wbytes;
        if (fa.nwin > 3) fa.nwin = 3;
        if (fa.nwin < 1) return DG_ERR_UNSUPPORTED;
        fa.fd_hpwp = cf_div((uint32_t)(Hp * Wp));
        fa.fd_wp = cf_div((uint32_t)Wp);
    }
    const int64_t nt = (int64_t)fa.ntp * fa.ntq;
    if (nt > INT32_MAX) return DG_ERR_SHAPE;
    fa.ntiles = (int32_t)nt;
    fa.direct = direct ? 1 : 0;
    fa.i2c = i2c ? 1 : 0;
    fa.X = x;
    fa.H = cv.H;
    fa.W = cv.W;
    int lg = 0;
    while ((1 << lg) < cb) ++lg;
    fa.Cb_log2 = lg;
    fa.kw = cv.kw;
    fa.kw_recip = (65536 + cv.kw - 1) / cv.kw;
    fa.stride = cv.stride;
    fa.pad = cv.pad;
    fa.Ho = cv.Ho;
    fa.Wo = cv.Wo;
    fa.kb = cv.kh * cv.kw * cb;
    fa.padsrc = cf_pad_source(cv.pad_code);
    if (!fa.padsrc) return DG_ERR_CUDA;
    fa.fd_wo = cf_div((uint32_t)cv.Wo);
    fa.fd_ho = cf_div((uint32_t)cv.Ho);
    fa.D = out;
    fa.ldd = ldd;
    fa.has_rq = rq ? 1 : 0;
    fa.early_b = (b_prepared && opt(OPT_EARLY_WEIGHTS)) ? 1 : 0;
    fa.omma = opt(OPT_F4_OMMA) ? 1 : 0;
    if (rq) {   // the 16-bit SIMD requant (reading Q23) is the only requant form of this kernel
        const int64_t *t = rq->thr;
        uint32_t m16 = 0, c16 = 0;
        if (!(acc_bound <= 32767 && t[0] > -((int64_t)1 << 30) && t[2] < ((int64_t)1 << 30) && (cout >> 1) <= CF_TAB_PAIRS &&
              opt(OPT_F16) && f16_params(t[0], t[1], t[2], m16, c16)))
            return DG_ERR_UNSUPPORTED;
        const int64_t thr0m1 = t[0] - 1;
        fa.f16_accmax = (int32_t)acc_bound;
        if (rq->bias) {   // per-column offsets, range-checked by the kernel when it builds their table
            fa.f16_tab = 1;
        } else {
            const int64_t n = -thr0m1;
            if ((n < 0 ? -n : n) + acc_bound > 32767) return DG_ERR_UNSUPPORTED;
            fa.f16_na2 = ((uint32_t)n & 0xFFFFu) * 0x10001u;
        }
        fa.f16_m = m16;
        fa.f16_c2 = c16 * 0x10001u;
        fa.f16_w2 = (uint32_t)(t[2] - t[0] + 1) * 0x10001u;
        fa.f16_thr0m1 = (int32_t)thr0m1;
    }
    CUtensorMap mp, mb;
    memset(&mp, 0, sizeof(mp));
    if (i2c) {
        if (!cf_map_im2col(&mp, x, cb, cv.W, cv.H, rows / ((int64_t)cv.Ho * cv.Wo), cv.stride)) return DG_ERR_CUDA;
    } else if (direct && !cf_map(&mp, x, cb, cb, rows, CF_BM)) {
        return DG_ERR_CUDA;
    }
    if (!cf_map(&mb, w4, ld4, ld4, cout, bnt)) return DG_ERR_CUDA;
    // (the shared-memory-A form, TA = false, measured 5-20 % slower: kept in the source, not built)
    const bool ta = true;
    // two CTAs per SM (option f4_ct = 2; 128-wide tiles): 4 unpack and 4 epilogue warps per CTA
    const int ct = (!win && bnt == 128 && opt(OPT_F4_CT) == 2) ? 2 : 1;
    const int nunp = (ct == 2) ? 4 : win ? 8 : ((int)opt(OPT_F4_UNP) == 4 ? 4 : ((int)opt(OPT_F4_UNP) == 8 ? 8 : (direct ? 4 : 8)));
    const int nepi = ct == 2 ? 4 : ((bnt == 64 || win) ? 8 : ((int)opt(OPT_F4_EPI) == 4 ? 4 : 8));   // (auto: 8, measured -5..-20 % on every FP4 layer)
    typedef void (*CfKern)(const CUtensorMap, const CUtensorMap, const CfArgs, const RequantArgs);
    static const CfKern kerns[25] = {
        lut_conv_f4_kernel<true, 4, 0, 128, 4, 1>, lut_conv_f4_kernel<true, 8, 0, 128, 4, 1>,
        lut_conv_f4_kernel<true, 4, 1, 128, 4, 1>,  lut_conv_f4_kernel<true, 8, 1, 128, 4, 1>,
        lut_conv_f4_kernel<true, 4, 0, 256, 4, 1>, lut_conv_f4_kernel<true, 8, 0, 256, 4, 1>,
        lut_conv_f4_kernel<true, 4, 1, 256, 4, 1>,  lut_conv_f4_kernel<true, 8, 1, 256, 4, 1>,
        lut_conv_f4_kernel<true, 4, 0, 128, 8, 1>, lut_conv_f4_kernel<true, 8, 0, 128, 8, 1>,
        lut_conv_f4_kernel<true, 4, 1, 128, 8, 1>,  lut_conv_f4_kernel<true, 8, 1, 128, 8, 1>,
        lut_conv_f4_kernel<true, 4, 0, 256, 8, 1>, lut_conv_f4_kernel<true, 8, 0, 256, 8, 1>,
        lut_conv_f4_kernel<true, 4, 1, 256, 8, 1>,  lut_conv_f4_kernel<true, 8, 1, 256, 8, 1>,
        lut_conv_f4_kernel<true, 4, 0, 128, 4, 2>, lut_conv_f4_kernel<true, 4, 1, 128, 4, 2>,
        lut_conv_f4_kernel<true, 4, 0, 64, 8, 1>,  lut_conv_f4_kernel<true, 8, 0, 64, 8, 1>,
        lut_conv_f4_kernel<true, 4, 1, 64, 8, 1>,   lut_conv_f4_kernel<true, 8, 1, 64, 8, 1>,
        lut_conv_f4_kernel<true, 8, 2, 64, 8, 1>,   lut_conv_f4_kernel<true, 8, 2, 128, 8, 1>,
        lut_conv_f4_kernel<true, 8, 2, 256, 8, 1>};
    static bool attr[25] = {};
    const int ai = win          ? (bnt == 64 ? 22 : bnt == 128 ? 23 : 24)
                   : ct == 2    ? 16 + (direct ? 1 : 0)
                   : bnt == 64 ? 18 + (direct ? 2 : 0) + (nunp == 8 ? 1 : 0)
                               : (nepi == 8 ? 8 : 0) + (bnt == 256 ? 4 : 0) + (direct ? 2 : 0) + (nunp == 8 ? 1 : 0);
    const CfKern kern = kerns[ai];
    if (!attr[ai]) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ct == 2 ? CF2_ALLOC : CF_ALLOC) !=
            cudaSuccess)
            return DG_ERR_CUDA;
        attr[ai] = true;
    }
    RequantArgs dummy{};
    const RequantArgs rqv = rq ? *rq : dummy;
    const int grid = (int)(nt < ct * num_sms() ? nt : ct * num_sms());
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)grid);
    lc.blockDim = dim3((unsigned)(32 * (3 + nepi + nunp)));
    lc.dynamicSmemBytes = ct == 2 ? CF2_ALLOC : CF_ALLOC;
    lc.stream = st;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = opt(OPT_PDL) ? 1 : 0;
    lc.attrs = la;
    lc.numAttrs = 1;
    if (cudaLaunchKernelEx(&lc, kern, mp, mb, fa, rqv) != cudaSuccess) return DG_ERR_CUDA;
    char tag[128];
    snprintf(tag, sizeof(tag), "f4conv bn=%d %s%s unp=%d epi=%d direct=%d%s rq=%d tab=%d early=%d omma=%d", bnt,
             win ? (fa.w1x1 ? "win1x1 wbres wpair " : fa.wpair ? "win wbres wpair " : fa.wbres ? "win wbres " : "win ") : "",
             ct == 2 ? "ta nacc=1 ct=2" : (bnt == 256 ? "ta nacc=1" : (bnt == 64 ? "ta nacc=4" : (win ? "ta nacc=3" : "ta nacc=2"))), nunp, nepi, fa.direct,
             fa.i2c ? " i2c" : "", fa.has_rq,
             fa.f16_tab, fa.early_b, fa.omma);
    set_last_kernel(tag);
    return launch_status();
}

}  // namespace dg
