// lut_gemm_ts.cu — the tensor-core LUT-16 GEMM for PRODUCT tables, "TS" form:
//
//   D[p][q] = sum_{k<K} pl[P[p][k]] * ql[Q[q][k]]  ==  sum_k T[(P<<2)|Q]      (Alg. 1)
//
// as a tcgen05 kind::i8 GEMM (exact s32 accumulation in TMEM) where
//   * the A operand (P, the packed 2-bit activations / im2col rows) is unpacked ON CHIP, one
//     thread per row, straight into TENSOR MEMORY with tcgen05.st (the paper's unpack step,
//     P:123, producing int8 levels): no shared-memory write of the 4x expanded data;
//   * the B operand (Q) is the int8 level expansion of the packed weights made ONCE by
//     dg_expand_operand (an offline weight transform, like the paper's offline weight packing
//     and reordering, P:143 / P:298), fed by TMA with the 128B swizzle into shared memory.
//
// Persistent, warp-specialised, one CTA per SM:
//   warps 0..3    epilogue: TMEM accumulators -> exact requant (S7) or int32 -> global
//   warps 4..11   unpackers: two groups of 4 warps (one warp per TMEM lane quarter) owning
//                 alternate stages; thread = row of the 128-row tile
//   warp 12       producer: packed P stages (128 B = 512 codes per row, TMA SWIZZLE_128B or a
//                 contiguous bulk copy when rows are <= 32 B) and int8 B stages (TMA, SW128)
//   warp 13       waiter: waits on the MMA-side mbarriers, hands stages to warp 14 by bar.sync
//   warp 14       MMA issuer (one thread): tcgen05.mma [D], [A_tmem], B_desc, 4 k-steps/stage
#include <cooperative_groups.h>
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "requant16.cuh"
#include "unpack.cuh"

namespace dg {
namespace {

constexpr int BM = 128;          // TMEM lanes / P rows per tile
constexpr int KA = 128;          // codes per B "atom": one 128-byte SW128 int8 row, 32 TMEM columns of A
constexpr int PKS_MAX = 128;     // packed bytes per row per packed slot (512 codes)
constexpr int TAB_PAIRS = 2048;  // per-column requant table (16-bit SIMD epilogue): nq <= 4096
constexpr int SP_MAX = 32;       // packed P slots (narrow rows -> many slots in flight)
// Warp roles.  The SM sub-partition scheduler prefers the highest warp id among eligible
// warps, so the latency-critical single-thread roles (TMA producer, MMA issuer) take the
// highest ids and are never starved by the ALU-heavy unpack / epilogue warps.
// NEPI (template) epilogue warps: 4 x EG groups; a group (one warp per TMEM lane quarter, all
// BN columns) owns every EG-th tile, so EG = 2 keeps two tiles' epilogues in flight (short-K
// tiles, where the epilogue dominates).
// NUNP (template) unpack warps: 4 (one stage group) or 8 (two groups owning alternate stages).
// EM (epilogue mode, template bits): EM_CSPLIT = every epilogue group works on every tile, group g on
// column block g (the accumulator is released as soon as each warp has loaded its columns) instead
// of groups owning alternate tiles; EM_HIGH = epilogue warps above the unpack warps in warp-id order
// (scheduler priority) for layers whose cost is the epilogue.
constexpr int EM_CSPLIT = 1, EM_HIGH = 2, EM_A6 = 4;
template <int NEPI, int NUNP, int EM = 0>
struct Roles {
    static constexpr int NUM_UGROUPS = NUNP / 4;
    static constexpr int EPI_WARP0 = (EM & EM_HIGH) ? NUNP : 0;          // lane quarter = warp % 4
    static constexpr int UNPACK_WARP0 = (EM & EM_HIGH) ? 0 : NEPI;        // lane quarter = warp % 4
    static constexpr int PRODUCER_WARP = NEPI + NUNP;
    static constexpr int WAITER_WARP = PRODUCER_WARP + 1;
    static constexpr int MMA_WARP = WAITER_WARP + 1;
    static constexpr int NT = 32 * (MMA_WARP + 1);
};
// An mbarrier probe (or any shared-memory load) issued by the warp that issues tcgen05.mma
// waits behind that warp's queued MMAs (measured ~670 cycles per probe, tools/mma_bench.cu),
// which drains the tensor pipe once per stage.  So the MMA warp never waits on an mbarrier:
// the waiter warp does, and hands each stage over with a named-barrier rendezvous, which does
// not stall the MMA queue (measured: 64 cycles per 128x128x32 MMA either way).
constexpr int HANDOFF_BAR = 1;
constexpr int EPI_BAR = 2;       // epilogue warps only (requant table build)

// KST (template): codes per pipeline stage, 128 or 256.  Every stage costs a fixed number of
// mbarrier / named-barrier hops (~150 cycles each, tools/sync_bench.cu) in the unpack, waiter and
// MMA roles, so long-K tiles use 256-code stages (8 MMAs of K = 32 per hand-off).
// WIN (template): direct 3x3 / stride-1 convolution.  The A operand is an unpacked window of
// padded input pixels in shared memory (no-swizzle K-major layout) and every tap's MMA reads it
// through a row-shifted descriptor, so each input pixel is unpacked once per tile instead of
// once per tap (im2col row).
// ASM (template): the A operand in SHARED memory (no-swizzle K-major stages written by the unpack
// warps, SS MMA) instead of tensor memory, which leaves all 512 TMEM columns to two 128x256
// accumulators: short-K, wide-output layers, whose cost is a fixed chain of hand-offs per tile.
template <int BN, int EG, int KST, bool WIN = false, bool ASM = false, bool A6 = false>
struct TsCfg {
    static constexpr int KSTEPS = KST / 32;                 // MMAs (K = 32) per stage
    static constexpr int ACOLS = KST / 4;                   // TMEM columns of one A stage
    static constexpr int HALVES = KST / KA;                 // 128-code halves (B atoms, 32-column A parts)
    // accumulator buffers (TMEM cols NACC*BN); a multiple of EG so that each buffer has one
    // epilogue group (which then waits on its barrier phases in order)
    // (ASM and WIN keep A in shared memory: all 512 TMEM columns hold accumulators)
    static constexpr int NACC = ASM ? 512 / BN : (WIN ? 4 : (BN == 256 ? 1 : (BN == 128 ? 2 : 4)));
    static_assert(NACC % EG == 0, "accumulator buffers per epilogue group");
    // (A6: the short-K shared-memory-A kernel with six A stages and at most two weight stages)
    static constexpr int SA = (ASM && A6) ? 6 : ((ASM || WIN) ? 4 : ((512 - NACC * BN) / ACOLS > 8 ? 8 : (512 - NACC * BN) / ACOLS));   // A stages (WIN: windows)
    static constexpr int B_ATOM = BN * KA;                  // bytes of one 128-code B atom
    static constexpr int B_BYTES = BN * KST;
    // WIN with 128-code stages = the C = 128 tile mode: all 9 weight stages (128 x 1152) resident
    static constexpr bool WIN128 = WIN && KST == 128;
    static constexpr int SB_RAW = (WIN128 ? 147456 : (WIN && BN == 64 ? 49152 : (BN == 64 || WIN || ASM ? 98304 : 131072))) / B_BYTES;
    static constexpr int SB_CAP = (ASM && A6) ? 2 : (WIN128 ? 9 : 8);
    static constexpr int SB = SB_RAW > SB_CAP ? SB_CAP : SB_RAW;   // B (int8) smem stages
    static constexpr int TMEM_A0 = NACC * BN;               // first A column
    static constexpr int TMEM_COLS = 512;
    static constexpr int P_REGION = WIN ? (WIN128 ? 70656 : (BN == 64 ? 155648 : 106496)) : (ASM ? 32768 : 4 * BM * PKS_MAX);   // packed P / WIN ring + windows
    static constexpr int A_STAGE = ASM ? BM * KST : 0;       // ASM: one A stage, 16-byte K chunk j of row r at j*BM*16 + r*16
    static constexpr int OFF_B = 0;                          // 1024-aligned (SW128)
    static constexpr int OFF_P = OFF_B + SB * B_BYTES;
    static constexpr int OFF_A = OFF_P + P_REGION;
    static constexpr int OFF_BAR = OFF_A + SA * A_STAGE;
    static constexpr int NBAR = 2 * SP_MAX + 2 * SB + 2 * SA + 2 * NACC;
    static constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
    static constexpr int OFF_WALK = OFF_TMEM + 16;           // 32 words: the MMA warp's copy of the tile walk
    static constexpr int OFF_OBAR = OFF_WALK + 128;          // offs: the offset block is ready (mbarrier)
    static constexpr int OFF_TAB = (OFF_OBAR + 16 + 15) / 16 * 16;   // 16-bit requant offsets, one u32 per column pair
    // int32-output staging for the TMA tensor store (4 epilogue warps x one 32 x 32 int32 chunk,
    // 128-byte swizzle, 1024-aligned) in the instances with one epilogue group and room for it
    static constexpr int STG_BYTES = (EG == 1 && !WIN && !ASM) ? 4 * 4096 : 0;
    static constexpr int OFF_STG = (OFF_TAB + TAB_PAIRS * 4 + 1023) / 1024 * 1024;
    // offs operands (no-swizzle K-major, 2 K chunks of 16 bytes): B rows per column tile (2 tiles),
    // then the constant A rows
    static constexpr int OFFS_BYTES = ASM ? 2 * BN * 32 + BM * 32 : 0;
    static constexpr int OFF_OFFS = (OFF_STG + STG_BYTES + 1023) / 1024 * 1024;
    static constexpr int ALLOC = OFF_OFFS + OFFS_BYTES + 1024;
    static_assert(((ASM || WIN) ? NACC * BN : TMEM_A0 + SA * ACOLS) <= TMEM_COLS && SA >= 2, "TMEM budget");
    static_assert(ALLOC <= 232448, "shared memory budget");
};

#ifdef DG_TRACE
// CTA 0 event timeline (tools/trace_ts.py): [event][stage or tile index] = clock(), recorded
// in shared memory (a global store per event perturbs the pipeline) and copied out at the end
constexpr int TL_N = 96, TL_E = 24;
__device__ long long g_ts_tl[TL_E][TL_N];
__shared__ uint32_t s_tl[TL_E][TL_N];
#define TS_EV(e, i) do { if ((int)(i) < TL_N) s_tl[e][i] = (uint32_t)clock(); } while (0)
#else
#define TS_EV(e, i) do { } while (0)
#endif

// n / d without a divide for 0 <= n < 2^31 (round-up multiplier; d >= 1):
// s = ceil(log2 d), m = floor(2^32 (2^s - d) / d) + 1, q = (umulhi(n, m) + n) >> s
struct FastDiv {
    uint32_t m, s;
};
inline FastDiv make_fastdiv(uint32_t d) {
    uint32_t s = 0;
    while ((1ull << s) < d) ++s;
    return FastDiv{(uint32_t)((((1ull << s) - d) << 32) / d + 1), s};
}
DG_DEV uint32_t fdiv(uint32_t n, FastDiv f) { return (__umulhi(n, f.m) + n) >> f.s; }

// tensor maps of the fused all-gather destinations (peer GPUs' C, P2P-mapped): the TMA-store
// epilogue writes every staged int32 chunk to its own C and, from the same shared-memory bytes,
// to each peer (whole 32 x 32 boxes per request instead of per-lane 16-byte stores)
struct PeerMaps {
    CUtensorMap m[7];
};

struct TsArgs {
    int64_t np, nq;
    int32_t nstages, last_ksteps, ntp, ntq;
    int32_t group;         // tile rasterisation: GROUP row blocks x all column blocks, column-major inside
    // split-K (few output tiles, long K): work item t = output tile t / sk, K stages of split t % sk;
    // each split stores its partial sums to its own slice ws_acc[ks] (int32 [sk][np][nq]); the
    // slices are summed and requantised / stored either by the same (cooperatively launched) kernel
    // after a grid-wide barrier (sk_fused: no second launch on the latency-bound chains) or by the
    // splitk_reduce_kernel launched right behind
    int32_t sk, nwork;   // nwork = ntp * ntq * sk work items
    int32_t sk_fused;
    // B multicast (bmc): CTA pairs of a 2-CTA cluster take row-adjacent tiles of the same column
    // block (the tile walk gives it when the grid, the raster group and the row-block count are
    // even); each CTA loads half of every B stage and multicasts it into both CTAs, and each MMA
    // warp's stage commit releases the slot in both (empty_b counts 2): half the L2 -> SM traffic
    // of the weights, which bounds the large GEMMs (no B reloads at all: 16384^3 3076 -> 3457 TOPS)
    int32_t bmc;
    // offs (short-K shared-memory-A instance, per-column requant offsets, <= 2 column tiles): each
    // tile's accumulator starts at its columns' 16-bit requant offsets n = bias - (t0 - 1) through
    // one extra K = 32 MMA (A rows [127, 1, 0...], B rows [q, r, 0...], n = 127 q + r), so the
    // epilogue's clamp takes no per-column offset loads (they were ~10 % of these layers)
    int32_t offs;
    // fused all-gather (int32 output): every output tile is also stored to npeer extra
    // destinations (peer GPUs' C buffers, P2P-mapped, already offset to this rank's rows)
    int32_t npeer;
    int32_t *peer[7];
    FastDiv fd_sk;
    int32_t *ws_acc;
    int32_t last_grp, last_rows;   // index of the last row group and its row-block count
    FastDiv fd_pg, fd_grp, fd_last;  // / (group * ntq), / group, / last_rows
    int32_t pks;           // packed P slot bytes per row (smem pitch): ldp <= 64 (bulk) or 128 (TMA box)
    int32_t bulk;          // 1: a tile's P rows are one contiguous span -> one bulk copy, unswizzled
    const uint8_t *P;
    int64_t ldp;
    int32_t sp;            // packed P slots (SP_MAX max)
    int32_t bres;          // 1: all ntq x nstages B tiles resident in smem (loaded once)
    int32_t early_b;       // 1: resident B tiles and the bias table are loaded before griddepcontrol.wait
    int32_t tma_d;         // 1: int32 output tiles leave through the TMA tensor store (tm_d, staging smem)
    uint32_t lp;           // int8 levels of P codes
    void *D;
    int64_t ldd;
    int32_t has_rq, fast_rq, dir;
    int32_t thr[3];
    // implicit-GEMM convolution: P = im2col of an NHWC packed input; every unpack thread gathers
    // its own row's taps with 16-byte cp.async copies IG_DEPTH stages ahead (group-private ring
    // in the packed-slot region)
    int32_t implicit;
    const uint8_t *X;      // [B][H][W][Cb] packed codes, Cb = C/4 a power of two >= 16
    int32_t H, W, Cb_log2, kw_recip, kw, stride, pad, Ho, Wo, kb;
    const uint8_t *padsrc; // 16 bytes of the pad code (out-of-image taps); padsrc + 16: zeros (beyond K)
    FastDiv fd_wo, fd_ho;
    // WIN (direct 3x3 conv): tiles run over the padded pixel space q = (b*Hp + hp)*Wp + wp
    // (Hp = H+2, Wp = W+2); window row i of a tile = padded pixel q0 - Wp - 1 + i
    int32_t win, Wp, WR, lbo, wslot, wbytes, nwin, clog2;   // WR window rows, lbo = WR*16
    int32_t wpair;         // WIN tile mode with 2 row blocks per work item (one window, 2 accumulators)
    int64_t nqv;           // B*Hp*Wp
    FastDiv fd_hpwp, fd_wp;
    uint16_t koff[72];     // A descriptor start offset (16-byte units) of k-step j: chunk and tap shift
    // 16-bit SIMD requant (host-verified, see f16_params): per column pair
    //   x = clamp(acc + negA, 0, W) (one VIADDMNMX.RELU), code = (x*m + c) >> 14 (one IMAD),
    // negA = bias - (thr0 - 1) per column (smem table), per row, or uniform.
    int32_t f16;           // 1: usable (all codes' thresholds finite, |acc| + |negA| < 2^15)
    int32_t f16_tab;       // 1: per-column bias -> negA table built in shared memory
    uint32_t f16_m, f16_c2, f16_w2, f16_na2;   // m; c and W replicated in both halves; uniform negA
    int32_t f16_thr0m1, f16_accmax;
    // residual in the 16-bit path (S7 with reading Q13): 1 = identity shortcut over packed codes,
    // r = res_levels[code]*res_mult (pair table res_pair[16] in smem); 2 = int32 residual
    // (downsample accumulators), packed to 16-bit pairs with a per-warp range check
    int32_t f16_res;
    uint32_t res_pair[16];    // (r[c0] & 0xFFFF) | r[c1] << 16 for the 4-bit pair index c0 | c1 << 2
};

// WIN "tile mode": C = 64 (18 k-steps of 32 codes = 9 taps x 2 chunks, stages 8 + 8 + 2) with the
// weights resident in shared memory, so a tile needs one hand-off and one burst of 18 MMAs
// (and C = 128 with 128-code stages: 36 k-steps = 9 taps x 4 chunks, 9 stages of 4)
DG_DEV bool win_tile_mode(const TsArgs &ta, int ksteps) {
    return ta.bres && !(ta.sk > 1) &&
           ((ta.clog2 == 6 && ksteps == 8 && ta.nstages == 3 && ta.last_ksteps == 2) ||
            (ta.clog2 == 7 && ksteps == 4 && ta.nstages == 9 && ta.last_ksteps == 4));
}

// Tile t -> (row block tp, column block tq).  Tiles are walked in groups of `group` row blocks,
// column block outer / row block inner, so that a wave of concurrent tiles touches few B tiles
// and few A row blocks (keeps a 256 MB int8 B operand from being re-streamed from HBM).
template <class A>
DG_DEV void tile_coords(const A &ta, int t, int &tp, int &tq) {
    const uint32_t grp = fdiv((uint32_t)t, ta.fd_pg);
    const uint32_t rem = (uint32_t)t - grp * (uint32_t)(ta.group * ta.ntq);
    const bool last = (int)grp == ta.last_grp;
    const uint32_t q = fdiv(rem, last ? ta.fd_last : ta.fd_grp);
    tq = (int)q;
    tp = (int)(grp * ta.group + (rem - q * (uint32_t)(last ? ta.last_rows : ta.group)));
}

// Work item t -> output tile (tp, tq) and its stages [sb, se) (all stages unless split-K)
// (SK: the kernel instance supports split-K; the others compile the plain tile walk)
template <bool SK, class A>
DG_DEV void work_item(const A &ta, int t, int &tp, int &tq, int &sb, int &se) {
    if (SK && ta.sk > 1) {
        const int ot = (int)fdiv((uint32_t)t, ta.fd_sk), ks = t - ot * ta.sk;
        tile_coords(ta, ot, tp, tq);
        sb = ks * ta.nstages / ta.sk;
        se = (ks + 1) * ta.nstages / ta.sk;
    } else {
        tile_coords(ta, t, tp, tq);
        sb = 0;
        se = ta.nstages;
    }
}

// The tile walk's parameters held in registers.  The MMA-issuing warp reads them through this
// copy: a parameter-space load (LDC) issued by that warp waits behind its queued MMAs, like a
// shared-memory load (measured on the WIN path: ~600 cycles per stage), so it must not touch
// the parameter struct between MMAs.
struct Walk {
    FastDiv fd_pg, fd_grp, fd_last, fd_sk;
    int32_t group, ntq, last_grp, last_rows, sk, nstages, bres, last_ksteps, ntiles, grid;
};
// The values are staged through shared memory and read back with volatile loads once, before
// the first MMA: ptxas would otherwise rematerialise them from the parameter bank inside the loop.
DG_DEV void put_walk(const TsArgs &ta, volatile uint32_t *d) {
    const uint32_t v[16] = {ta.fd_pg.m, ta.fd_pg.s, ta.fd_grp.m, ta.fd_grp.s, ta.fd_last.m, ta.fd_last.s, ta.fd_sk.m,
                            ta.fd_sk.s, (uint32_t)ta.group, (uint32_t)ta.ntq, (uint32_t)ta.last_grp,
                            (uint32_t)ta.last_rows, (uint32_t)ta.sk, (uint32_t)ta.nstages, (uint32_t)ta.bres,
                            (uint32_t)ta.last_ksteps};
    for (int i = 0; i < 16; ++i) d[i] = v[i];
    d[16] = (uint32_t)ta.nwork;
    d[17] = gridDim.x;
}
DG_DEV Walk get_walk(const volatile uint32_t *d) {
    uint32_t v[18];
#pragma unroll
    for (int i = 0; i < 18; ++i) v[i] = d[i];
    Walk w;
    w.fd_pg = FastDiv{v[0], v[1]};
    w.fd_grp = FastDiv{v[2], v[3]};
    w.fd_last = FastDiv{v[4], v[5]};
    w.fd_sk = FastDiv{v[6], v[7]};
    w.group = (int32_t)v[8];
    w.ntq = (int32_t)v[9];
    w.last_grp = (int32_t)v[10];
    w.last_rows = (int32_t)v[11];
    w.sk = (int32_t)v[12];
    w.nstages = (int32_t)v[13];
    w.bres = (int32_t)v[14];
    w.last_ksteps = (int32_t)v[15];
    w.ntiles = (int32_t)v[16];
    w.grid = (int32_t)v[17];
    return w;
}

// Implicit im2col gather cursor of one unpack thread (row r of its tiles): walks the thread's
// group's stages (every NUM_UGROUPS-th stage across tiles) and issues each stage's 16-byte chunks
// (64 codes each) as cp.async copies into one slot of the group's ring.  K order (r, s, c) with c
// fastest (dg_im2col); out-of-image taps copy the pad code, bytes beyond K copy zeros.
template <bool SK>
struct GatherCursor {
    int t, s;                 // work item and (absolute) stage of the next fetch
    const uint8_t *img;
    int32_t h0, w0;
    int se;                   // end of the work item's stage range
    DG_DEV void pixel(const TsArgs &ta, int r) {
        int tp, tq, sb;
        work_item<SK>(ta, t, tp, tq, sb, se);
        const int64_t p = (int64_t)tp * BM + r;
        const uint32_t pp = (uint32_t)(p < ta.np ? p : ta.np - 1);
        const uint32_t tt = fdiv(pp, ta.fd_wo), b = fdiv(tt, ta.fd_ho);
        img = ta.X + (((int64_t)b * ta.H * ta.W) << ta.Cb_log2);
        h0 = (int32_t)(tt - b * (uint32_t)ta.Ho) * ta.stride - ta.pad;
        w0 = (int32_t)(pp - tt * (uint32_t)ta.Wo) * ta.stride - ta.pad;
    }
    DG_DEV void advance(const TsArgs &ta, int by, int r, int ntiles) {
        s += by;
        if constexpr (!SK) {
            bool moved = false;
            while (s >= ta.nstages) { s -= ta.nstages; t += gridDim.x; moved = true; }
            if (moved && t < ntiles) pixel(ta, r);
        } else {
            while (s >= se && t < ntiles) {   // into the next work item of this CTA
                const int over = s - se;
                t += gridDim.x;
                if (t >= ntiles) break;
                pixel(ta, r);   // sets se
                int tp, tq, sb, se2;
                work_item<SK>(ta, t, tp, tq, sb, se2);
                s = sb + over;
            }
        }
    }
    template <int NCH>
    DG_DEV void issue(const TsArgs &ta, uint32_t dst_row, int r, int ntiles, int bytes_per_stage) {
        if (t < ntiles) {
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                const int32_t byte = s * bytes_per_stage + 16 * c;
                const int32_t tap = byte >> ta.Cb_log2;
                const int32_t off = byte & ((1 << ta.Cb_log2) - 1);
                const int32_t rr = (tap * ta.kw_recip) >> 16;   // tap / kw (exact for kh*kw <= 64)
                const int32_t ss = tap - rr * ta.kw;
                const int32_t hi = h0 + rr, wi = w0 + ss;
                const uint8_t *src = byte >= ta.kb ? ta.padsrc + 16
                                     : ((uint32_t)hi < (uint32_t)ta.H && (uint32_t)wi < (uint32_t)ta.W)
                                           ? img + ((((int64_t)hi * ta.W + wi) << ta.Cb_log2) + off)
                                           : ta.padsrc;
                // 64-byte row pitch, 16-byte unit c at c ^ ((r >> 1) & 3): conflict-free LDS.128
                ptx::cp_async16(dst_row + ((c ^ ((r >> 1) & 3)) << 4), src);
            }
        }
        ptx::cp_async_commit();
    }
};

// int32 output / residual requant / ragged tail for one 32-column chunk of accumulator values
__device__ __forceinline__ void ts_epilogue_values(const TsArgs &ta, const RequantArgs &rq, const int32_t (&v)[32], int64_t p,
                                                int64_t qc) {
    if (p >= ta.np || qc >= ta.nq) return;
    if (!ta.has_rq) {
        const bool vec = qc + 32 <= ta.nq && (ta.ldd & 3) == 0 && ((reinterpret_cast<uintptr_t>(ta.D) & 15) == 0);
        for (int d = -1; d < ta.npeer; ++d) {   // own output, then the all-gather peers (same offsets)
            int32_t *dp = (d < 0 ? reinterpret_cast<int32_t *>(ta.D) : ta.peer[d]) + p * ta.ldd + qc;
            if (vec) {
#pragma unroll
                for (int j = 0; j < 32; j += 4) *reinterpret_cast<int4 *>(dp + j) = make_int4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            } else {
                for (int j = 0; j < 32; ++j)
                    if (qc + j < ta.nq) dp[j] = v[j];
            }
        }
        return;
    }
    uint8_t *dp = reinterpret_cast<uint8_t *>(ta.D) + p * ta.ldd + (qc >> 2);
    if (qc + 32 <= ta.nq) {
        const uint2 o = requant_row32(rq, v, p, qc);
        if ((reinterpret_cast<uintptr_t>(dp) & 7) == 0) *reinterpret_cast<uint2 *>(dp) = o;
        else store_codes32_ts(dp, o.x, o.y, 8);
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
    store_codes32_ts(dp, o0, o1, (int)((ta.nq - qc + 3) / 4));
}

// the same from tensor memory (warp-collective load)
__device__ __noinline__ void ts_epilogue_general(const TsArgs &ta, const RequantArgs &rq, uint32_t taddr, int64_t p,
                                                 int64_t qc) {
    uint32_t rr[32];
    ptx::tmem_ld_32x32b_x32(taddr, rr);
    ptx::tmem_ld_wait();
    int32_t v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = (int32_t)rr[j];
    ts_epilogue_values(ta, rq, v, p, qc);
}

// split-K partial tile: this split's accumulators go to its own slice ws_acc[ks][np][nq]; each
// lane writes whole 128-byte row segments (measured: scattered int32 atomics into one shared
// partial, or a last-arriver reduction by the 32-lane quarter that owns the rows, both cost more
// than the split saved — the reduction is latency-bound per lane; a separate grid-wide reduce
// kernel is one round trip)
__device__ __noinline__ void ts_epilogue_splitk(const TsArgs &ta, uint32_t trow, int nch, int64_t p, int64_t q0, int ks,
                                                int lane, uint32_t acc_bar) {
    const bool vec = (ta.nq & 3) == 0;
    int32_t *row = ta.ws_acc + ks * ta.np * ta.nq + p * ta.nq;
    for (int c = 0; c < nch; ++c) {
        uint32_t rr[32];
        ptx::tmem_ld_32x32b_x32(trow + c * 32, rr);
        ptx::tmem_ld_wait();
        if (c == nch - 1) {   // the accumulator buffer is free again
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(acc_bar);
        }
        const int64_t qc = q0 + c * 32;
        if (p >= ta.np || qc >= ta.nq) continue;
        if (vec && qc + 32 <= ta.nq) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
                __stcg(reinterpret_cast<int4 *>(row + qc + j),
                       make_int4((int32_t)rr[j], (int32_t)rr[j + 1], (int32_t)rr[j + 2], (int32_t)rr[j + 3]));
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (qc + j < ta.nq) __stcg(row + qc + j, (int32_t)rr[j]);
        }
    }
}

// split-K reduction: one thread per (row p, 4 consecutive columns): sum the sk <= 8 slices (all
// loads in flight at once), then requantise to one byte of codes (4 columns, LSB first; columns
// past nq give zero bits, as the fused epilogue writes them) or store the int32 sums.
DG_DEV void splitk_reduce_range(const int32_t *__restrict__ ws, int64_t np, int64_t nq, int32_t sk, void *D, int64_t ldd,
                                int32_t has_rq, const RequantArgs &rq, int64_t i0, int64_t di) {
    const int64_t ng = (nq + 3) >> 2, n = np * ng, slice = np * nq;
    const bool vec = (nq & 3) == 0;
    for (int64_t i = i0; i < n; i += di) {
        const int64_t p = i / ng, q = (i - p * ng) * 4;
        const int32_t *src = ws + p * nq + q;
        int32_t v[4] = {0, 0, 0, 0};
        if (vec) {
            int4 t[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) t[k] = k < sk ? __ldcg(reinterpret_cast<const int4 *>(src + k * slice)) : make_int4(0, 0, 0, 0);
#pragma unroll
            for (int k = 0; k < 8; ++k) { v[0] += t[k].x; v[1] += t[k].y; v[2] += t[k].z; v[3] += t[k].w; }
        } else {
            for (int k = 0; k < sk; ++k)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (q + j < nq) v[j] += __ldcg(src + k * slice + j);
        }
        if (!has_rq) {
            int32_t *dp = reinterpret_cast<int32_t *>(D) + p * ldd + q;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (q + j < nq) dp[j] = v[j];
        } else {
            uint32_t b = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (q + j < nq) b |= requant_one(rq, v[j], p, q + j) << (2 * j);
            reinterpret_cast<uint8_t *>(D)[p * ldd + (q >> 2)] = (uint8_t)b;
        }
    }
}

__global__ void __launch_bounds__(256) splitk_reduce_kernel(const int32_t *__restrict__ ws, int64_t np, int64_t nq,
                                                            int32_t sk, void *D, int64_t ldd, int32_t has_rq,
                                                            RequantArgs rq) {
    ptx::griddep_wait();   // the split-K GEMM's slices are complete and visible
    splitk_reduce_range(ws, np, nq, sk, D, ldd, has_rq, rq, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                        (int64_t)gridDim.x * blockDim.x);
}

// 16-bit SIMD requant of one tile (S7): RES = 0 no residual, 1 identity shortcut over packed
// codes (pair table in smem), 2 int32 residual (exact redo of a chunk where |r| >= 2^14).  The
// residual forms are compiled out of the RES = 0 instance (they cost registers / spills there).
// TAB: per-column offsets from the shared-memory table, else one offset per row (na_row); a
// runtime branch here made the compiler merge the two na[] arrays with ~64 register moves per
// 32 columns (measured 8% of the K = 64 layers' instructions).
template <int BN, int RES, bool TAB>
__device__ __forceinline__ void epi16_tile(const TsArgs &ta, const RequantArgs &rq, uint32_t trow, int64_t p, int64_t q0,
                                           uint32_t na_row, uint32_t tab, int lane, uint32_t acc_bar, uint32_t tl_ev = 0) {
    constexpr int NCH = BN / 32;
    // all of the tile's accumulators (up to 128 columns as 16-bit pairs) are loaded
    // before any requant work, so the TMEM buffer goes back to the MMA as early as
    // possible (the accumulator ring is only NACC = 2 deep for 128-column tiles)
    constexpr int NLD = NCH / 2 < 2 ? NCH / 2 : 2;   // 64-column loads held in registers
#pragma unroll 1
    for (int c0 = 0; c0 < NCH; c0 += 2 * NLD) {
        uint32_t r16[NLD][32];
#pragma unroll
        for (int l = 0; l < NLD; ++l) ptx::tmem_ld_32x32b_x32_pack16(trow + (c0 + 2 * l) * 32, r16[l]);
        ptx::tmem_ld_wait();
        if (lane == 0 && threadIdx.x < 32) TS_EV(c0 == 0 ? 16 : 18, tl_ev);
        if (c0 + 2 * NLD >= NCH && RES != 2) {   // (int32 residual: kept for an exact redo)
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(acc_bar);
        }
#ifdef DG_EXP_LDONLY
        if (r16[0][5] != 0x12345u) continue;
#endif
#pragma unroll
        for (int hh = 0; hh < 2 * NLD; ++hh) {
            const int64_t qc = q0 + (c0 + hh) * 32;
            uint32_t na[16];
#ifdef DG_EXP_NOLDS
            if (false) {
#else
            if constexpr (TAB) {
#endif
                const uint32_t ta4 = tab + (uint32_t)(qc >> 1) * 4u;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint4 t4 = ptx::lds128(ta4 + 16 * j);
                    na[4 * j] = t4.x; na[4 * j + 1] = t4.y; na[4 * j + 2] = t4.z; na[4 * j + 3] = t4.w;
                }
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) na[j] = na_row;
            }
            uint32_t rr[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) rr[j] = r16[hh >> 1][16 * (hh & 1) + j];
            if constexpr (RES == 1) {   // identity shortcut: pair residuals from the packed codes
                const uint2 rc = p < ta.np ? *reinterpret_cast<const uint2 *>(rq.res_codes + p * rq.ld_res_codes + (qc >> 2))
                                           : make_uint2(0, 0);
                const uint32_t rt = tab + 4u * (TAB_PAIRS - 16);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    uint32_t rp;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(rp) : "r"(rt + 4u * (((j < 8 ? rc.x : rc.y) >> (4 * (j & 7))) & 15u)));
                    rr[j] = __vadd2(rr[j], rp);
                }
            } else if constexpr (RES == 2) {   // int32 residual -> 16-bit pairs (|r| < 2^14 checked)
                uint32_t bad = 0;
                if (p < ta.np) {
                    const int4 *rp = reinterpret_cast<const int4 *>(rq.res + p * rq.ld_res + qc);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int4 v = __ldg(rp + j);
                        bad |= (uint32_t)(v.x + 16384) | (uint32_t)(v.y + 16384) | (uint32_t)(v.z + 16384) | (uint32_t)(v.w + 16384);
                        rr[2 * j] = __vadd2(rr[2 * j], prmt_b32((uint32_t)v.x, (uint32_t)v.y, 0x5410u));
                        rr[2 * j + 1] = __vadd2(rr[2 * j + 1], prmt_b32((uint32_t)v.z, (uint32_t)v.w, 0x5410u));
                    }
                }
                if (__any_sync(0xFFFFFFFFu, (bad >> 15) != 0u)) {   // exact redo of this chunk (TMEM still held)
                    ts_epilogue_general(ta, rq, trow + (uint32_t)((c0 + hh) * 32), p, qc);
                    continue;
                }
            }
            if (p >= ta.np) continue;
            const uint2 o = requant16_32(rr, na, ta.f16_w2, ta.f16_m, ta.f16_c2);
            uint8_t *dp = reinterpret_cast<uint8_t *>(ta.D) + p * ta.ldd + (qc >> 2);
#ifdef DG_EXP_NOSTORE
            if (o.x == 0x12345678u && o.y == 0x9abcdef0u)
#endif
            if ((reinterpret_cast<uintptr_t>(dp) & 7) == 0) *reinterpret_cast<uint2 *>(dp) = o;
            else store_codes32_ts(dp, o.x, o.y, 8);
        }
        if (lane == 0 && threadIdx.x < 32) TS_EV(c0 == 0 ? 17 : 19, tl_ev);
    }
    if constexpr (RES == 2) {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(acc_bar);
    }
}

// Epilogue tile loop for the launch-uniform rare modes — split-K partial tiles, and 16-bit
// requant with a residual — kept out of line: inlined, their code raised register pressure in the
// common loop past the 128-register cap and its spills cost ~40% on short-K layers (measured).
template <int BN, int NACC, int EG, bool WIN, bool CS>
__device__ __noinline__ void epilogue_loop_rare(const TsArgs &ta, const RequantArgs &rq, uint32_t tmem, uint32_t tab,
                                                uint32_t acc_bar0, int ntiles, int warp, int lane, bool f16_ok) {
    // CS: group eg takes columns [eg * BN / EG, (eg + 1) * BN / EG) of every tile
    constexpr int CW = CS ? BN / EG : BN, NCH = CW / 32;
    const int quarter = warp & 3, eg = warp >> 2;
    uint32_t tl = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
        if (!CS && EG > 1 && (int)(tl % EG) != eg) continue;
        const uint32_t acc = tl % NACC;
        const uint32_t acc_full = acc_bar0 + 8 * acc, acc_empty = acc_bar0 + 8 * (NACC + acc);
        int tp, tq, sb_, se_;
        work_item<true>(ta, t, tp, tq, sb_, se_);
        const int64_t p = (int64_t)tp * BM + quarter * 32 + lane;
        const int64_t q0 = (int64_t)tq * BN + (CS ? eg * CW : 0);
        ptx::mbar_wait(acc_full, (tl / NACC) & 1u);
        ptx::tc_fence_after();
        const uint32_t trow = tmem + acc * BN + (CS ? eg * CW : 0) + ((uint32_t)(quarter * 32) << 16);
        if (ta.sk > 1) {
            ts_epilogue_splitk(ta, trow, NCH, p, q0, (int)(t - (int)fdiv((uint32_t)t, ta.fd_sk) * ta.sk), lane, acc_empty);
            continue;
        }
        // residual in the 16-bit path (every lane's row offset must fit int16 for bias_axis 1)
        bool use16 = f16_ok && q0 + CW <= ta.nq;
        uint32_t na_row = ta.f16_na2;
        if (use16 && !ta.f16_tab && rq.bias && rq.bias_axis == 1) {
            const int64_t n = (int64_t)(p < ta.np ? __ldg(rq.bias + p) : 0) - ta.f16_thr0m1;
            na_row = ((uint32_t)n & 0xFFFFu) * 0x10001u;
            use16 = __all_sync(0xFFFFFFFFu, (n < 0 ? -n : n) + ta.f16_accmax <= 32767);
        }
        if (use16 && ta.f16_res == 1) {
            if (ta.f16_tab) epi16_tile<CW, 1, true>(ta, rq, trow, p, q0, na_row, tab, lane, acc_empty);
            else epi16_tile<CW, 1, false>(ta, rq, trow, p, q0, na_row, tab, lane, acc_empty);
        } else if (use16 && ta.f16_res == 2) {
            if (ta.f16_tab) epi16_tile<CW, 2, true>(ta, rq, trow, p, q0, na_row, tab, lane, acc_empty);
            else epi16_tile<CW, 2, false>(ta, rq, trow, p, q0, na_row, tab, lane, acc_empty);
        } else {
#pragma unroll 1
            for (int c = 0; c < NCH; ++c) ts_epilogue_general(ta, rq, trow + c * 32, p, q0 + c * 32);
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(acc_empty);
        }
    }
}

template <int BN, int NEPI, int NUNP, int KST, bool WIN, bool ASM, bool SK, int EM>
__global__ void __launch_bounds__(Roles<NEPI, NUNP, EM>::NT, 1)
lut_gemm_ts_kernel(const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_b,
                   const __grid_constant__ CUtensorMap tm_d, const __grid_constant__ PeerMaps pm,
                   const __grid_constant__ TsArgs ta, const __grid_constant__ RequantArgs rq,
                   const __grid_constant__ CUtensorMap tm_bh) {   // tm_bh: B boxes of BN / 2 rows (bmc)
    using C = TsCfg<BN, (EM & EM_CSPLIT) ? 1 : NEPI / 4, KST, WIN, ASM, (EM & EM_A6) != 0>;
    using R = Roles<NEPI, NUNP, EM>;
    constexpr bool CS = (EM & EM_CSPLIT) != 0;
    constexpr int SB = C::SB, SA = C::SA, NACC = C::NACC, SP = SP_MAX;
    const int nsp = ta.sp;
    const uint32_t pslot = (uint32_t)(BM * ta.pks);
    constexpr int NUM_EPI_WARPS = NEPI, EPI_WARP0 = R::EPI_WARP0, UNPACK_WARP0 = R::UNPACK_WARP0,
                  PRODUCER_WARP = R::PRODUCER_WARP, WAITER_WARP = R::WAITER_WARP, MMA_WARP = R::MMA_WARP,
                  NUM_UGROUPS = R::NUM_UGROUPS;
    extern __shared__ uint8_t smem_raw[];
#ifdef DG_TRACE
    for (int i = threadIdx.x; i < TL_E * TL_N; i += blockDim.x) (&s_tl[0][0])[i] = 0u;
#endif
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = ptx::smem_u32(smem);
    const uint32_t bar0 = sbase + C::OFF_BAR;
    auto full_p = [&](int s) { return bar0 + 8 * s; };
    auto empty_p = [&](int s) { return bar0 + 8 * (SP + s); };
    auto full_b = [&](int s) { return bar0 + 8 * (2 * SP + s); };
    auto empty_b = [&](int s) { return bar0 + 8 * (2 * SP + SB + s); };
    auto full_a = [&](int s) { return bar0 + 8 * (2 * SP + 2 * SB + s); };
    auto empty_a = [&](int s) { return bar0 + 8 * (2 * SP + 2 * SB + SA + s); };
    auto acc_full = [&](int a) { return bar0 + 8 * (2 * SP + 2 * SB + 2 * SA + a); };
    auto acc_empty = [&](int a) { return bar0 + 8 * (2 * SP + 2 * SB + 2 * SA + NACC + a); };
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + C::OFF_TMEM);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntiles = ta.nwork;   // work items (split-K: sk per output tile; a param-space operand, never spilled)
    const int nsub = (ta.pks * 4 + KST - 1) / KST;   // stages per packed slot

    if (warp == PRODUCER_WARP) {
        if (lane == 0) {
            if (!ta.implicit && !ta.bulk) ptx::tma_prefetch(&tm_p);
            ptx::tma_prefetch(&tm_b);
            for (int s = 0; s < SP; ++s) {
                ptx::mbar_init(full_p(s), 1);
                ptx::mbar_init(empty_p(s), nsub * 4);   // 4 warps (one group) per stage, nsub stages
            }
            for (int s = 0; s < SB; ++s) {
                ptx::mbar_init(full_b(s), 1);
                ptx::mbar_init(empty_b(s), ta.bmc ? 2 : 1);   // (bmc: both CTAs' MMA commits)
            }
            for (int s = 0; s < SA; ++s) {   // WIN: window buffers, filled by all unpack warps
                ptx::mbar_init(full_a(s), WIN ? NUNP : 4);
                ptx::mbar_init(empty_a(s), 1);
            }
            for (int a = 0; a < NACC; ++a) {
                ptx::mbar_init(acc_full(a), 1);
                ptx::mbar_init(acc_empty(a), CS ? NEPI : 4);   // the 4 warps of the owning group (CS: all)
            }
            if (ASM && ta.offs) ptx::mbar_init(sbase + C::OFF_OBAR, NEPI);   // every epilogue warp's offsets written
            ptx::fence_mbar_init();
        }
        __syncwarp();
        ptx::tmem_alloc(ptx::smem_u32(tmem_slot), C::TMEM_COLS);
    }
    uint32_t *f16tab = reinterpret_cast<uint32_t *>(smem + C::OFF_TAB);
    volatile uint32_t *f16_flag = reinterpret_cast<volatile uint32_t *>(smem + C::OFF_TMEM + 8);
    volatile uint32_t *offs_bad = reinterpret_cast<volatile uint32_t *>(smem + C::OFF_OBAR + 8);
    if (threadIdx.x == 0) {
        *f16_flag = 0u;
        *offs_bad = 0u;
        *reinterpret_cast<volatile uint32_t *>(smem + C::OFF_TMEM + 12) = 0u;   // the MMA warp's opaque zero
        put_walk(ta, reinterpret_cast<volatile uint32_t *>(smem + C::OFF_WALK));
    }
    // (with __syncthreads_or here the kernel faulted with a misaligned address when launched
    // right after the tc_ss kernel, cause not determined: the flag goes through shared memory)
    ptx::tc_fence_before();
    __syncthreads();
    if (ta.bmc) ptx::cluster_sync_all();   // the partner's barriers are initialised before any multicast
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // programmatic dependent launch: the next layer's CTAs may start (prologue) as ours exit; every
    // role waits for the previous grid before touching activations / outputs (weights and the
    // requant table are set-up data and are read before the wait)
    if (threadIdx.x == 0) ptx::griddep_launch_dependents();

    if (warp == PRODUCER_WARP) {
        // ---------------- producer.  The whole warp runs the loop (a lone lane 0 with 31 lanes
        // parked at the final __syncthreads ran the loop several times slower); lane 0 issues.
        uint32_t gb = 0, pslot_i = 0, pphase = 0;
        // (the B operand may have been written by the previous kernel on the stream, e.g. the weight
        // expansion of dg_lut_conv2d: only the early_weights contract lets it be read before the wait)
        if (!ta.bres || !ta.early_b) ptx::griddep_wait();
        if (ta.bres) {   // every B tile once: slot tq * nstages + s
            for (int tq = 0; tq < ta.ntq; ++tq)
                for (int s = 0; s < ta.nstages; ++s) {
                    const int j = tq * ta.nstages + s;
                    if (lane == 0) {
                        ptx::mbar_arrive_expect_tx(full_b(j), (uint32_t)C::B_BYTES);
#pragma unroll
                        for (int h = 0; h < C::HALVES; ++h)
                            ptx::tma_load_2d(sbase + C::OFF_B + j * C::B_BYTES + h * C::B_ATOM, &tm_b, full_b(j),
                                             s * KST + h * KA, tq * BN);
                    }
                }
            __syncwarp();
            if (ta.early_b) ptx::griddep_wait();
        }
        // the loop's parameters in registers (warp shuffles: ptxas cannot rematerialise them from
        // the parameter bank inside the loop)
        const Walk wk = get_walk(reinterpret_cast<volatile uint32_t *>(smem + C::OFF_WALK));
        const bool p_load = !WIN && ptx::opaque((uint32_t)ta.implicit) == 0u;
        const bool p_bulk = ptx::opaque((uint32_t)ta.bulk) != 0u, p_bres = ptx::opaque((uint32_t)ta.bres) != 0u,
                   p_bmc = ptx::opaque((uint32_t)ta.bmc) != 0u;
        const int64_t p_np = (int64_t)ptx::opaque64((uint64_t)ta.np), p_ldp = (int64_t)ptx::opaque64((uint64_t)ta.ldp);
        const uint8_t *p_src = reinterpret_cast<const uint8_t *>(ptx::opaque64(reinterpret_cast<uint64_t>(ta.P)));
        const int p_pks = (int)ptx::opaque((uint32_t)ta.pks), p_nsub = (int)ptx::opaque((uint32_t)nsub),
                  p_nsp = (int)ptx::opaque((uint32_t)nsp);
        const uint32_t p_slot = ptx::opaque(pslot);
        const int p_ntl = wk.ntiles, p_grid = wk.grid;
        int t_first = blockIdx.x;
        if (p_load && p_bres && wk.nstages == 1) {
            // one-slot tiles with resident weights (the short-K 1x1 layers): the loop is a chain of
            // dependent instructions (~900 cycles per tile measured, tools/trace_ts.py --prod), the
            // pace of the whole pipeline.  Lane i < PB takes the round's i-th tile: its coordinates,
            // slot wait and copy issue run side by side with the other lanes'
            const int PB = p_nsp < 8 ? p_nsp : 8;
            for (int t0 = blockIdx.x; t0 < p_ntl; t0 += PB * p_grid) {
                const int t = t0 + lane * p_grid;
                const int cnt = (p_ntl - t0 + p_grid - 1) / p_grid < PB ? (p_ntl - t0 + p_grid - 1) / p_grid : PB;
                if (lane < cnt) {
                    int tp, tq, sb, se;
                    work_item<SK>(wk, t, tp, tq, sb, se);
                    const int64_t p0 = (int64_t)tp * BM;
                    const uint32_t li = pslot_i + (uint32_t)lane;
                    const bool wrap = li >= (uint32_t)p_nsp;
                    const int slot = (int)(wrap ? li - (uint32_t)p_nsp : li);
                    ptx::mbar_wait(empty_p(slot), (pphase ^ (wrap ? 1u : 0u)) ^ 1u);
                    const uint32_t dst = sbase + C::OFF_P + (uint32_t)slot * p_slot;
                    if (p_bulk) {
                        const int64_t rows = p_np - p0 < BM ? p_np - p0 : BM;
                        const uint32_t bytes = (uint32_t)(rows * p_ldp);
                        ptx::mbar_arrive_expect_tx(full_p(slot), bytes);
                        ptx::bulk_load(dst, p_src + p0 * p_ldp, bytes, full_p(slot));
                    } else {
                        ptx::mbar_arrive_expect_tx(full_p(slot), p_slot);
                        ptx::tma_load_2d(dst, &tm_p, full_p(slot), 0, (int32_t)p0);
                    }
                }
                __syncwarp();
                pslot_i += (uint32_t)cnt;
                if (pslot_i >= (uint32_t)p_nsp) { pslot_i -= (uint32_t)p_nsp; pphase ^= 1u; }
                gb += (uint32_t)cnt;
            }
            t_first = p_ntl;
        }
        for (int t = t_first; t < p_ntl; t += p_grid) {
            int tp, tq, sb, se;
            work_item<SK>(wk, t, tp, tq, sb, se);
            if (lane == 0) TS_EV(23, gb);
            const int64_t p0 = (int64_t)tp * BM, q0 = (int64_t)tq * BN;
            int sub = 0, ps = 0;
            for (int s = sb; s < se; ++s, ++gb) {
                if (sub == 0 && p_load) {   // next packed P slot (up to 512 codes of every row)
                    const int slot = (int)pslot_i;
                    if (lane == 0) TS_EV(13, gb);
                    ptx::mbar_wait(empty_p(slot), pphase ^ 1u);
                    if (lane == 0) {
                        TS_EV(14, gb);
                        const uint32_t dst = sbase + C::OFF_P + slot * p_slot;
                        if (p_bulk) {   // (a TMA box of narrow rows issues one request per row: slow)
                            const int64_t rows = p_np - p0 < BM ? p_np - p0 : BM;
                            const uint32_t bytes = (uint32_t)(rows * p_ldp);
                            ptx::mbar_arrive_expect_tx(full_p(slot), bytes);
                            ptx::bulk_load(dst, p_src + p0 * p_ldp, bytes, full_p(slot));
                        } else {
                            ptx::mbar_arrive_expect_tx(full_p(slot), p_slot);
                            ptx::tma_load_2d(dst, &tm_p, full_p(slot), sb * (KST / 4) + ps * p_pks, (int32_t)p0);
                        }
                        TS_EV(12, gb);
                    }
                    __syncwarp();
                    if (lane == 0) TS_EV(22, gb);
                    if (++pslot_i == (uint32_t)p_nsp) { pslot_i = 0; pphase ^= 1u; }
                    ++ps;
                }
                if (++sub == p_nsub) sub = 0;
                if (p_bres) continue;
                const int bs = gb % SB;
                ptx::mbar_wait(empty_b(bs), ((gb / SB) & 1u) ^ 1u);
                if (lane == 0) {
                    ptx::mbar_arrive_expect_tx(full_b(bs), (uint32_t)C::B_BYTES);   // (bmc: both halves land here)
                    if (p_bmc) {
                        const uint32_t rk = ptx::cluster_ctarank();
#pragma unroll
                        for (int h = 0; h < C::HALVES; ++h)
                            ptx::tma_load_2d_multicast(sbase + C::OFF_B + bs * C::B_BYTES + h * C::B_ATOM + rk * (C::B_ATOM / 2),
                                                       &tm_bh, full_b(bs), s * KST + h * KA, (int32_t)(q0 + rk * (BN / 2)), 0x3);
                    } else {
#pragma unroll
                        for (int h = 0; h < C::HALVES; ++h)
                            ptx::tma_load_2d(sbase + C::OFF_B + bs * C::B_BYTES + h * C::B_ATOM, &tm_b, full_b(bs),
                                             s * KST + h * KA, (int32_t)q0);
                    }
                }
                __syncwarp();
            }
        }
    } else if (warp == WAITER_WARP) {
        // ---------------- waiter: acc_empty / full_a / full_b, then rendezvous with the MMA warp
        ptx::griddep_wait();
        // resident B: wait for all of it once (each mbarrier probe costs ~150 cycles even when the
        // phase completed long ago, and the waiter's probes are on the critical path of short tiles)
        if (ta.bres)
            for (int j = 0; j < ta.ntq * ta.nstages; ++j) ptx::mbar_wait(full_b(j), 0u);
        uint32_t g = 0, tl = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
            const uint32_t u0 = WIN ? (tl << ta.wpair) : tl;   // accumulator use index (WIN pairs: 2 per item)
            if (NACC > 1) ptx::mbar_wait(acc_empty(u0 % NACC), ((u0 / NACC) & 1u) ^ 1u);   // (NACC 1: the MMA warp)
            int tp, tq, sb, se;
            work_item<SK>(ta, t, tp, tq, sb, se);
            if (WIN) ptx::mbar_wait(full_a(tl % ta.nwin), (tl / ta.nwin) & 1u);   // the tile's window
            if (WIN && lane == 0) TS_EV(13, tl);
            if (WIN && win_tile_mode(ta, C::KSTEPS)) {   // one hand-off per tile (B resident)
                if (ta.wpair) ptx::mbar_wait(acc_empty((u0 + 1) % NACC), (((u0 + 1) / NACC) & 1u) ^ 1u);
                ptx::named_bar_sync(HANDOFF_BAR, 64);
                g += (uint32_t)(se - sb);
                continue;
            }
            for (int s = sb; s < se; ++s, ++g) {
                const int sa = g % SA;
                if (lane == 0 && s == sb) TS_EV(3, tl);
                if (!WIN) ptx::mbar_wait(full_a(sa), (g / SA) & 1u);
                if (lane == 0) TS_EV(4, g);
                if (!ta.bres) ptx::mbar_wait(full_b(g % SB), (g / SB) & 1u);
                if (lane == 0) TS_EV(5, g);
                ptx::named_bar_sync(HANDOFF_BAR, 64);
                if (lane == 0) TS_EV(6, g);   // the MMA warp finished issuing stage g - 1
            }
        }
    } else if (warp == MMA_WARP) {
        // ---------------- MMA issuer: no mbarrier waits here (see HANDOFF_BAR).  The whole warp runs
        // the loop and the *_warp helpers elect the issuing lane inside their asm (ptx::mma_i8_ts_warp).
        constexpr uint32_t idesc = ptx::idesc_i8(BM, BN);
        const uint64_t bdesc0 = ptx::desc_k_sw128(sbase + C::OFF_B);
        // parameters in registers before any MMA is queued (Walk)
        const uint32_t z0 = *reinterpret_cast<volatile uint32_t *>(smem + C::OFF_TMEM + 12);   // 0
        auto reg_copy = [z0](uint32_t x) { return x + z0; };
        // WIN geometry in registers before any MMA is queued
        const int w_slot = (int)reg_copy((uint32_t)ta.wslot), w_nwin = (int)reg_copy((uint32_t)ta.nwin),
                  w_bytes = (int)reg_copy((uint32_t)ta.wbytes);
        const uint32_t w_lbo16 = reg_copy((uint32_t)ta.lbo >> 4), w_wp = reg_copy((uint32_t)ta.Wp),
                       w_clog2 = reg_copy((uint32_t)ta.clog2);
        const int w_pair = WIN ? (int)reg_copy((uint32_t)ta.wpair) : 0;
        // offs: wait once for the epilogue warps' offset rows; the same flags decide their epilogue form
        bool w_offs = false;
        if (ASM && reg_copy((uint32_t)ta.offs) != 0u) {
            ptx::mbar_wait(sbase + C::OFF_OBAR, 0u);
            w_offs = *f16_flag == 0u && *offs_bad == 0u;
        }
        const uint64_t one_desc = ptx::desc_k_none(sbase + C::OFF_OFFS + 2 * BN * 32, BM * 16);
        const bool w_bmc = !WIN && !ASM && reg_copy((uint32_t)ta.bmc) != 0u;   // commits release both CTAs' B slot
        uint32_t w_tap[9];   // window row shift of tap (r, s) in 16-byte units: r*Wp + s
#pragma unroll
        for (int q = 0; q < 9; ++q) w_tap[q] = (uint32_t)(q / 3) * w_wp + (uint32_t)(q % 3);
        const Walk wk = get_walk(reinterpret_cast<volatile uint32_t *>(smem + C::OFF_WALK));
        const bool win_mode = WIN && win_tile_mode(ta, C::KSTEPS);
        const int ntl = wk.ntiles, grid_n = wk.grid;
        uint32_t g = 0, tl = 0;
        for (int t = blockIdx.x; t < ntl; t += grid_n, ++tl) {
            const uint32_t acc = tl % NACC;
            const uint32_t dt = tmem + acc * BN;
            int tp, tq, sb, se;
            work_item<SK>(wk, t, tp, tq, sb, se);
            if (WIN && win_mode) {
                // C = 64 direct 3x3 with resident weights: the tile's 18 k-steps (tap j/2, channel
                // chunk 2(j&1)) issued after one hand-off, with compile-time B offsets and the 9 tap
                // offsets of the window held in registers (no per-stage hand-off, no memory op).
                // Pair mode: the window spans 2 row blocks; block h reads it BM rows further down
                // and accumulates into the next accumulator buffer.
                const uint32_t wbase = sbase + C::OFF_P + (uint32_t)(2 * w_slot + (int)(tl % w_nwin) * w_bytes);
                const uint64_t ad = ptx::desc_k_none(wbase, w_lbo16 << 4);
                const uint64_t bt = bdesc0 + (uint64_t)((tq * (KST == 256 ? 3 : 9) * C::B_BYTES) >> 4);
                ptx::named_bar_sync(HANDOFF_BAR, 64);
                ptx::tc_fence_after();
                if (lane == 0) TS_EV(14, g);
                for (int h = 0; h <= w_pair; ++h) {
                    const uint32_t u = (tl << w_pair) + (uint32_t)h;
                    const uint32_t dth = tmem + (u % NACC) * BN;
                    const uint64_t adh = ad + (uint64_t)(h * BM);   // BM rows of 16 bytes
                    // k-step j: tap j / (C/32), channel chunk 2 (j mod C/32); B stage j / KSTEPS
                    constexpr int CPT = KST == 256 ? 2 : 4;   // k-steps per tap (C = 64 / 128)
#pragma unroll
                    for (int j = 0; j < 9 * CPT; ++j) {
                        const int st = j / C::KSTEPS, k = j % C::KSTEPS;
                        ptx::mma_i8_ss_warp(dth, adh + (uint64_t)(w_tap[j / CPT] + (uint32_t)((j % CPT) * 2) * w_lbo16),
                                            bt + (uint64_t)((st * C::B_BYTES + (k >> 2) * C::B_ATOM) >> 4) + 2 * (k & 3),
                                            idesc, j > 0 ? 1u : 0u);
                    }
                    ptx::mma_commit_warp(acc_full(u % NACC));
                }
                ptx::mma_commit_warp(empty_a(tl % w_nwin));   // the window is free again
                if (lane == 0) TS_EV(15, g);
                g += (uint32_t)(se - sb);
                __syncwarp();
                continue;
            }
            // a single accumulator (128 x 256 tiles) is waited for here, in parallel with the waiter's
            // operand waits; with several, the MMA warp must not block (its mbarrier probes wait
            // behind its queued MMAs), the waiter takes them
            if (NACC == 1) ptx::mbar_wait(acc_empty(0), (tl & 1u) ^ 1u);
            for (int s = sb; s < se; ++s, ++g) {
                const int sa = g % SA;
                const int bsl = wk.bres ? tq * wk.nstages + s : (int)(g % SB);   // B smem stage
                const int nk = (s < wk.nstages - 1) ? C::KSTEPS : wk.last_ksteps;
                const uint64_t bd = bdesc0 + (uint64_t)((bsl * C::B_BYTES) >> 4);
                // WIN: k = tap*C + c: A = the window shifted by r*Wp + s rows (tap = 3r + s), K chunk
                // c/16; the per-k-step descriptors (host-precomputed offsets ta.koff) are formed before
                // the hand-off, so that no parameter load sits between two tcgen05.mma (a load there
                // serialises the issue: ~150 cycles per MMA measured)
                uint64_t wad[C::KSTEPS];
                if (WIN) {
                    const uint32_t wbase = sbase + C::OFF_P + (uint32_t)(2 * w_slot + (int)(tl % w_nwin) * w_bytes);
                    const uint64_t ad = ptx::desc_k_none(wbase, w_lbo16 << 4);
                    const int j0 = s * C::KSTEPS;
                    // k-step j (32 codes): tap = 32j / C, channel chunk (32j mod C) / 16, tap (r, s) =
                    // (tap / 3, tap mod 3) -> start offset chunk*lbo + (r*Wp + s)*16 bytes (the
                    // host's ta.koff, recomputed here with ALU ops only: an indexed parameter load
                    // in this warp waits for its queued MMAs)
#pragma unroll
                    for (int k = 0; k < C::KSTEPS; ++k) {
                        const uint32_t kb = (uint32_t)(32 * (j0 + k));
                        const uint32_t tap = kb >> w_clog2, chunk = (kb & ((1u << w_clog2) - 1u)) >> 4;
                        const uint32_t rr = (tap * 11u) >> 5;   // tap / 3 for tap < 9
                        wad[k] = ad + (uint64_t)(chunk * w_lbo16 + rr * w_wp + (tap - 3u * rr));
                    }
                }
                if (lane == 0) TS_EV(13, g);
                ptx::named_bar_sync(HANDOFF_BAR, 64);
                if (lane == 0) TS_EV(7, g);
                ptx::tc_fence_after();
                if (lane == 0) TS_EV(14, g);
                if (WIN) {
                    if (nk == C::KSTEPS) {   // full stage: straight-line issue
#pragma unroll
                        for (int k = 0; k < C::KSTEPS; ++k)
                            ptx::mma_i8_ss_warp(dt, wad[k], bd + (uint64_t)(((k >> 2) * C::B_ATOM) >> 4) + 2 * (k & 3),
                                                idesc, (s > sb || k > 0) ? 1u : 0u);
                    } else {
                        for (int k = 0; k < nk; ++k)
                            ptx::mma_i8_ss_warp(dt, wad[k], bd + (uint64_t)(((k >> 2) * C::B_ATOM) >> 4) + 2 * (k & 3),
                                                idesc, (s > sb || k > 0) ? 1u : 0u);
                    }
                    if (!wk.bres) ptx::mma_commit_warp(empty_b(bsl));
                    if (s == se - 1) {
                        ptx::mma_commit_warp(empty_a(tl % w_nwin));   // the window is free again
                        ptx::mma_commit_warp(acc_full(acc));
                    }
                } else if (ASM) {
                    const uint64_t ad = ptx::desc_k_none(sbase + C::OFF_A + (uint32_t)(sa * C::A_STAGE), BM * 16);
                    // offs: the tile's first MMA writes the columns' requant offsets into the accumulator
                    if (w_offs && s == sb)
                        ptx::mma_i8_ss_warp(dt, one_desc, ptx::desc_k_none(sbase + C::OFF_OFFS + (uint32_t)(tq * BN * 32), BN * 16),
                                            idesc, 0u);
                    // k-step k: A K-chunks 2k, 2k+1 (+2k * BM*16 bytes), B atom k/4, +32 B per k-step inside
                    if (nk == C::KSTEPS) {
#pragma unroll
                        for (int k = 0; k < C::KSTEPS; ++k)
                            ptx::mma_i8_ss_warp(dt, ad + (uint64_t)((2 * k * BM * 16) >> 4),
                                                bd + (uint64_t)(((k >> 2) * C::B_ATOM) >> 4) + 2 * (k & 3), idesc,
                                                (w_offs || s > sb || k > 0) ? 1u : 0u);
                    } else {
                        for (int k = 0; k < nk; ++k)
                            ptx::mma_i8_ss_warp(dt, ad + (uint64_t)((2 * k * BM * 16) >> 4),
                                                bd + (uint64_t)(((k >> 2) * C::B_ATOM) >> 4) + 2 * (k & 3), idesc,
                                                (w_offs || s > sb || k > 0) ? 1u : 0u);
                    }
                    ptx::mma_commit_warp(empty_a(sa));
                    if (!wk.bres) ptx::mma_commit_warp(empty_b(bsl));
                    if (s == se - 1) ptx::mma_commit_warp(acc_full(acc));
                } else {
                    const uint32_t at = tmem + C::TMEM_A0 + sa * C::ACOLS;
                    // k-step k: A columns 8k, B atom k/4 (+B_ATOM bytes), 32 bytes (+2) per k-step inside
#ifndef DG_EXP_NOMMA
                    if (nk == C::KSTEPS) {   // full stage: straight-line issue
#pragma unroll
                        for (int k = 0; k < C::KSTEPS; ++k)
                            ptx::mma_i8_ts_warp(dt, at + 8 * k, bd + (uint64_t)(((k >> 2) * C::B_ATOM) >> 4) + 2 * (k & 3),
                                                idesc, (s > sb || k > 0) ? 1u : 0u);
                    } else {
                        for (int k = 0; k < nk; ++k)
                            ptx::mma_i8_ts_warp(dt, at + 8 * k, bd + (uint64_t)(((k >> 2) * C::B_ATOM) >> 4) + 2 * (k & 3),
                                                idesc, (s > sb || k > 0) ? 1u : 0u);
                    }
#endif
                    ptx::mma_commit_warp(empty_a(sa));
                    if (w_bmc) ptx::mma_commit_warp_multicast(empty_b(bsl), 0x3);
                    else if (!wk.bres) ptx::mma_commit_warp(empty_b(bsl));
                    if (s == se - 1) ptx::mma_commit_warp(acc_full(acc));
                }
                if (lane == 0) TS_EV(15, g);
                __syncwarp();
            }
        }
    } else if (warp >= UNPACK_WARP0 && warp < UNPACK_WARP0 + NUNP && WIN) {
        // ---------------- WIN: fill each tile's window of padded input pixels.  Thread = window row:
        // its packed pixel (C/4 bytes) arrives by cp.async two tiles ahead (ring of 2 slots), is
        // unpacked to int8 levels and stored as C/16 16-byte K chunks (chunk j at j*lbo + row*16).
        ptx::griddep_wait();
        constexpr int WRING = 2;
        const int tid = (warp - UNPACK_WARP0) * 32 + lane;
        const bool has_row = tid < ta.WR;
        const int cb = 1 << (ta.clog2 - 2), nch = cb >> 4;   // packed bytes per pixel, 16-byte chunks
        const uint32_t ring = sbase + C::OFF_P, wins = ring + WRING * ta.wslot;
        // wide images (window > one row per thread, C = 64 only): thread tid owns rows tid + i*NUNP*32
        constexpr int WMAXR = 3;
        const int nrt = (ta.WR + NUNP * 32 - 1) / (NUNP * 32);
        // window row -> source pixel, in 32-bit arithmetic (host: B (H+2)(W+2) < 2^31 and the NHWC byte
        // offsets < 2^31): the fill warps' address chains paced the C = 64 layers (trace: ~1200 cycles
        // of each fill's ~2400 went to this fetch with 64-bit index math)
        const uint32_t w_hpwp = (uint32_t)((ta.H + 2) * ta.Wp), w_nqv = (uint32_t)ta.nqv, w_wp = (uint32_t)ta.Wp;
        const uint32_t w_h = (uint32_t)ta.H, w_w = (uint32_t)ta.W, w_sh = (uint32_t)(ta.clog2 - 2);
        auto fetch = [&](int t, int slot) {
            if (t < ntiles) {
                int tp, tq;
                tile_coords(ta, t, tp, tq);
                const uint32_t q0 = ((uint32_t)tp << ta.wpair) * BM - (w_wp + 1u);   // (wraps for the first rows)
                for (int i = 0; i < nrt; ++i) {
                    const int row = tid + i * NUNP * 32;
                    if (row >= ta.WR) break;
                    const uint32_t q = q0 + (uint32_t)row;   // padded pixel of this row
                    const uint8_t *src = ta.padsrc;
                    uint32_t step = 0;
                    if (q < w_nqv) {
                        const uint32_t b = fdiv(q, ta.fd_hpwp);
                        const uint32_t rem = q - b * w_hpwp;
                        const uint32_t hp = fdiv(rem, ta.fd_wp), wp = rem - hp * w_wp;
                        if (hp - 1u < w_h && wp - 1u < w_w) {
                            src = ta.X + (((b * w_h + hp - 1u) * w_w + wp - 1u) << w_sh);
                            step = 16;
                        }
                    }
                    const uint32_t dst = ring + (uint32_t)(slot * ta.wslot + row * cb);
                    for (int c = 0; c < nch; ++c) ptx::cp_async16(dst + 16 * c, src + c * step);
                }
            }
            ptx::cp_async_commit();
        };
        fetch(blockIdx.x, 0);
        fetch(blockIdx.x + gridDim.x, 1);
        uint32_t tl = 0;
        if (nrt > 1 && nch == 2) {   // C = 128 (two 16-byte chunks per row), up to 2 rows per thread
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
                const int slot = (int)(tl & 1u), wb = (int)(tl % ta.nwin);
                ptx::cp_async_wait<WRING - 1>();
                uint32_t a[2][32];
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int row = tid + i * NUNP * 32;
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const uint4 v = (i < nrt && row < ta.WR) ? ptx::lds128(ring + (uint32_t)(slot * ta.wslot + row * cb + 16 * c))
                                                                 : make_uint4(0, 0, 0, 0);
                        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint4 o = unpack16_levels(w[q], ta.lp);
                            a[i][16 * c + 4 * q] = o.x; a[i][16 * c + 4 * q + 1] = o.y;
                            a[i][16 * c + 4 * q + 2] = o.z; a[i][16 * c + 4 * q + 3] = o.w;
                        }
                    }
                }
                fetch(t + 2 * (int)gridDim.x, slot);   // the slot's bytes are consumed: refill it
                ptx::mbar_wait(empty_a(wb), ((tl / ta.nwin) & 1u) ^ 1u);   // the window's previous tile finished
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int row = tid + i * NUNP * 32;
                    if (i >= nrt || row >= ta.WR) break;
                    const uint32_t wdst = wins + (uint32_t)(wb * ta.wbytes + row * 16);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(wdst + (uint32_t)(j * ta.lbo)),
                                     "r"(a[i][4 * j]), "r"(a[i][4 * j + 1]), "r"(a[i][4 * j + 2]), "r"(a[i][4 * j + 3])
                                     : "memory");
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(full_a(wb));
            }
        } else if (nrt > 1) {   // (host guarantees C = 64: one 16-byte chunk per row)
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
                const int slot = (int)(tl & 1u), wb = (int)(tl % ta.nwin);
                ptx::cp_async_wait<WRING - 1>();
                uint32_t a[WMAXR][16];
#pragma unroll
                for (int i = 0; i < WMAXR; ++i) {
                    const int row = tid + i * NUNP * 32;
                    const uint4 v = (i < nrt && row < ta.WR) ? ptx::lds128(ring + (uint32_t)(slot * ta.wslot + row * cb))
                                                             : make_uint4(0, 0, 0, 0);
                    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint4 o = unpack16_levels(w[q], ta.lp);
                        a[i][4 * q] = o.x; a[i][4 * q + 1] = o.y; a[i][4 * q + 2] = o.z; a[i][4 * q + 3] = o.w;
                    }
                }
                fetch(t + 2 * (int)gridDim.x, slot);   // the slot's bytes are consumed: refill it
                ptx::mbar_wait(empty_a(wb), ((tl / ta.nwin) & 1u) ^ 1u);   // the window's previous tile finished
#pragma unroll
                for (int i = 0; i < WMAXR; ++i) {
                    const int row = tid + i * NUNP * 32;
                    if (i >= nrt || row >= ta.WR) break;
                    const uint32_t wdst = wins + (uint32_t)(wb * ta.wbytes + row * 16);
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(wdst + (uint32_t)(j * ta.lbo)),
                                     "r"(a[i][4 * j]), "r"(a[i][4 * j + 1]), "r"(a[i][4 * j + 2]), "r"(a[i][4 * j + 3])
                                     : "memory");
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(full_a(wb));
            }
        } else
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
            const int slot = (int)(tl & 1u), wb = (int)(tl % ta.nwin);
            if (tid == 0) TS_EV(0, tl);
            ptx::cp_async_wait<WRING - 1>();
            if (tid == 0) TS_EV(12, tl);
            uint32_t a[64];
            const uint32_t src = ring + (uint32_t)(slot * ta.wslot + tid * cb);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if (c >= nch) break;
                const uint4 v = has_row ? ptx::lds128(src + 16 * c) : make_uint4(0, 0, 0, 0);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint4 o = unpack16_levels(w[i], ta.lp);
                    a[16 * c + 4 * i] = o.x; a[16 * c + 4 * i + 1] = o.y; a[16 * c + 4 * i + 2] = o.z; a[16 * c + 4 * i + 3] = o.w;
                }
            }
            fetch(t + 2 * (int)gridDim.x, slot);   // the slot's bytes are consumed: refill it
            if (tid == 0) TS_EV(1, tl);
            ptx::mbar_wait(empty_a(wb), ((tl / ta.nwin) & 1u) ^ 1u);   // the window's previous tile finished
            if (tid == 0) TS_EV(11, tl);
            if (has_row) {
                const uint32_t wdst = wins + (uint32_t)(wb * ta.wbytes + tid * 16);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (j >= 4 * nch) break;
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(wdst + (uint32_t)(j * ta.lbo)),
                                 "r"(a[4 * j]), "r"(a[4 * j + 1]), "r"(a[4 * j + 2]), "r"(a[4 * j + 3])
                                 : "memory");
                }
            }
            ptx::fence_proxy_async_smem();   // generic-proxy stores -> visible to the tensor core
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(full_a(wb));
            if (tid == 0) TS_EV(2, tl);
        }
    } else if (warp >= UNPACK_WARP0 && warp < UNPACK_WARP0 + NUNP) {
        // ---------------- unpackers: thread = row; packed smem -> int8 levels -> TMEM (A operand).
        // Groups of 4 warps (one per TMEM lane quarter) take alternate stages.
        ptx::griddep_wait();
        const int uw = warp - UNPACK_WARP0;
        const int grp = uw / 4;                 // stage group
        const int quarter = warp & 3;           // TMEM lane quarter this warp may access
        const int r = quarter * 32 + lane;      // tile row
        const uint32_t trow_a = tmem + C::TMEM_A0 + ((uint32_t)(quarter * 32) << 16);
        const uint32_t msk = ta.bulk ? 0u : 7u;
        uint32_t g = 0, pslot_i = 0, pphase = 0;
        // implicit conv: group-private ring of IG_DEPTH stages (64 bytes per row each)
        constexpr int IG_DEPTH = C::P_REGION / (NUM_UGROUPS * BM * 64);
        const uint32_t ring = sbase + C::OFF_P + (uint32_t)(grp * IG_DEPTH * BM * 64) + (uint32_t)(r * 64);
        GatherCursor<SK> gc{(int)blockIdx.x, 0, ta.X, 0, 0, 0};
        uint32_t consumed = 0;
        if (KST == 128 && ta.nstages == 1 && !ta.implicit) {
            // one-stage tiles (K <= 128): a group unpacks two of its tiles per round of mbarrier
            // hand-offs (each hop ~150 cycles, tools/sync_bench.cu), halving the per-tile chain
            const int nch = (ta.last_ksteps + 1) / 2;   // 16-byte chunks read (1 or 2)
            for (uint32_t tl0 = grp; blockIdx.x + tl0 * gridDim.x < (uint32_t)ntiles; tl0 += 2 * NUM_UGROUPS) {
                const uint32_t tl1 = tl0 + NUM_UGROUPS;
                const bool has1 = blockIdx.x + tl1 * gridDim.x < (uint32_t)ntiles;
                if (lane == 0 && quarter == 0) TS_EV(0, tl0);
                uint4 v[2][2];
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    const uint32_t tl = b ? tl1 : tl0;
                    if (b && !has1) break;
                    const int slot = (int)(tl % (uint32_t)nsp);
                    ptx::mbar_wait(full_p(slot), (tl / (uint32_t)nsp) & 1u);
                    const uint32_t pbase = sbase + C::OFF_P + slot * pslot, lin = (uint32_t)(r * ta.pks);
                    v[b][0] = ptx::lds128(pbase + (lin ^ (((lin >> 7) & msk) << 4)));
                    v[b][1] = nch > 1 ? ptx::lds128(pbase + ((lin + 16) ^ ((((lin + 16) >> 7) & msk) << 4))) : make_uint4(0, 0, 0, 0);
                }
                uint32_t a[2][32];
#pragma unroll
                for (int b = 0; b < 2; ++b)
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        if (c >= nch) break;
                        const uint32_t w[4] = {v[b][c].x, v[b][c].y, v[b][c].z, v[b][c].w};
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const uint4 o = unpack16_levels(w[i], ta.lp);
                            a[b][16 * c + 4 * i] = o.x; a[b][16 * c + 4 * i + 1] = o.y; a[b][16 * c + 4 * i + 2] = o.z;
                            a[b][16 * c + 4 * i + 3] = o.w;
                        }
                    }
                // the slots are released only once their loaded values are USED: an mbarrier arrive
                // does not wait for outstanding shared-memory loads, and the TMA / bulk copy that
                // refills a slot after the arrive can overtake them (measured on the FP4 conv kernel)
                {
                    const uint32_t dep = v[0][0].x ^ v[0][1].x ^ v[1][0].x ^ v[1][1].x;
                    ptx::release_after_loads(empty_p((int)(tl0 % (uint32_t)nsp)), (uint32_t)nsub, dep);
                    if (has1) ptx::release_after_loads(empty_p((int)(tl1 % (uint32_t)nsp)), (uint32_t)nsub, dep);
                }
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    const uint32_t tl = b ? tl1 : tl0;
                    if (b && !has1) break;
                    const int sa = (int)(tl % SA);
                    ptx::mbar_wait(empty_a(sa), ((tl / SA) & 1u) ^ 1u);   // MMA(tl - SA) completed
                    if (ASM) {   // shared-memory A stage: K chunk j (16 codes) of row r at j*BM*16 + r*16
                        const uint32_t ab = sbase + C::OFF_A + (uint32_t)(sa * C::A_STAGE) + (uint32_t)(r * 16);
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            if (j >= 4 * nch) break;
                            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(ab + (uint32_t)(j * BM * 16)),
                                         "r"(a[b][4 * j]), "r"(a[b][4 * j + 1]), "r"(a[b][4 * j + 2]), "r"(a[b][4 * j + 3]) : "memory");
                        }
                    } else {
                        ptx::tc_fence_after();
                        if (nch > 1) ptx::tmem_st_32x32b_x32(trow_a + sa * C::ACOLS, a[b]);
                        else ptx::tmem_st_32x32b_x16(trow_a + sa * C::ACOLS, a[b]);
                    }
                }
                if (ASM) ptx::fence_proxy_async_smem();   // generic stores -> visible to the tensor core
                else ptx::tmem_st_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    ptx::mbar_arrive(full_a((int)(tl0 % SA)));
                    if (has1) ptx::mbar_arrive(full_a((int)(tl1 % SA)));
                }
                if (lane == 0 && quarter == 0) { TS_EV(2, tl0); TS_EV(2, tl1); }
            }
        } else {
        if (ta.implicit) {
            if (gc.t < ntiles) {   // first work item: start at its first stage, then this group's offset
                gc.pixel(ta, r);
                int tp, tq, sb, se2;
                work_item<SK>(ta, gc.t, tp, tq, sb, se2);
                gc.s = sb;
            }
            gc.advance(ta, grp, r, ntiles);
            for (int i = 0; i < IG_DEPTH; ++i) {
                gc.issue<2 * C::HALVES>(ta, ring + (uint32_t)(i * BM * 64), r, ntiles, KST / 4);
                gc.advance(ta, NUM_UGROUPS, r, ntiles);
            }
        }
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            int sub = 0, tp_, tq_, sb, se;
            work_item<SK>(ta, t, tp_, tq_, sb, se);
            for (int s = sb; s < se; ++s, ++g) {
                const int slot = (int)pslot_i;
                const uint32_t ph = pphase;
                const int sub_ = sub;
                const bool last_in_slot = (sub == nsub - 1) || (s == se - 1);
                if (last_in_slot) {
                    sub = 0;
                    if (++pslot_i == (uint32_t)nsp) { pslot_i = 0; pphase ^= 1u; }
                } else {
                    ++sub;
                }
                if ((int)(g % NUM_UGROUPS) != grp) continue;
                const int sa = g % SA;
                // 16-byte chunks (64 codes, 2 k-steps) of this stage that the MMA reads
                const int nchunk = (s != ta.nstages - 1) ? 2 * C::HALVES : (ta.last_ksteps + 1) / 2;
                if (lane == 0 && quarter == 0) TS_EV(0, g);
                uint4 v[2 * C::HALVES];
                if (ta.implicit) {
                    ptx::cp_async_wait<IG_DEPTH - 1>();   // this stage's copies (the oldest group) landed
                    const uint32_t row = ring + (uint32_t)((consumed % IG_DEPTH) * BM * 64);
#pragma unroll
                    for (int c = 0; c < 2 * C::HALVES; ++c)
                        v[c] = c < nchunk ? ptx::lds128(row + ((c ^ ((r >> 1) & 3)) << 4)) : make_uint4(0, 0, 0, 0);
                } else {
                    ptx::mbar_wait(full_p(slot), ph);
                    if (lane == 0 && quarter == 0) TS_EV(20, g);
                    // TMA slots carry the 128-byte swizzle: the 16-byte unit (bits 4-6) of the
                    // slot's linear offset is XORed with bits 7-9 (conflict-free LDS.128)
                    const uint32_t pbase = sbase + C::OFF_P + slot * pslot;
                    const uint32_t lin0 = (uint32_t)(r * ta.pks + sub_ * (KST / 4));
#pragma unroll
                    for (int c = 0; c < 2 * C::HALVES; ++c) {
                        const uint32_t lin = lin0 + 16 * c;
                        v[c] = c < nchunk ? ptx::lds128(pbase + (lin ^ (((lin >> 7) & msk) << 4))) : make_uint4(0, 0, 0, 0);
                    }
                }
                // unpack the whole stage into registers before waiting for the A buffer, so that the
                // wait overlaps the ALU work (a[32 h + j]: 32-column half h)
                uint32_t a[32 * C::HALVES];
#pragma unroll
                for (int c = 0; c < 2 * C::HALVES; ++c) {
                    if (c >= nchunk) break;
                    const uint32_t w[4] = {v[c].x, v[c].y, v[c].z, v[c].w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint4 o = unpack16_levels(w[i], ta.lp);
                        a[16 * c + 4 * i] = o.x; a[16 * c + 4 * i + 1] = o.y; a[16 * c + 4 * i + 2] = o.z;
                        a[16 * c + 4 * i + 3] = o.w;
                    }
                }
                if (lane == 0 && quarter == 0) TS_EV(21, g);
                if (ta.implicit) {   // the ring slot's data is consumed (values in registers): refill it
                    gc.issue<2 * C::HALVES>(ta, ring + (uint32_t)((consumed % IG_DEPTH) * BM * 64), r, ntiles, KST / 4);
                    gc.advance(ta, NUM_UGROUPS, r, ntiles);
                    ++consumed;
                } else {   // this warp's share of the slot is consumed (+ the slot's unused stages); released
                           // only after the values are used (see the one-stage path above)
                    uint32_t dep = 0;
#pragma unroll
                    for (int c = 0; c < 2 * C::HALVES; ++c) dep ^= v[c].x;
                    ptx::release_after_loads(empty_p(slot), 1u + (s == se - 1 ? (uint32_t)(nsub - 1 - sub_) : 0u), dep);
                }
                if (lane == 0 && quarter == 0) TS_EV(1, g);
                ptx::mbar_wait(empty_a(sa), ((g / SA) & 1u) ^ 1u);   // MMA(g - SA) completed
                if (lane == 0 && quarter == 0) TS_EV(11, g);
                ptx::tc_fence_after();
                if (ASM) {   // shared-memory A stage: K chunk j (16 codes) of row r at j*BM*16 + r*16
                    const uint32_t ab = sbase + C::OFF_A + (uint32_t)(sa * C::A_STAGE) + (uint32_t)(r * 16);
#pragma unroll
                    for (int j = 0; j < 8 * C::HALVES; ++j) {
                        if (j >= 4 * nchunk) break;
                        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(ab + (uint32_t)(j * BM * 16)),
                                     "r"(a[4 * j]), "r"(a[4 * j + 1]), "r"(a[4 * j + 2]), "r"(a[4 * j + 3]) : "memory");
                    }
                    ptx::fence_proxy_async_smem();
                } else {
#pragma unroll
                for (int h = 0; h < C::HALVES; ++h) {
                    if (2 * h >= nchunk) break;
                    uint32_t ah[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) ah[j] = a[32 * h + j];
#ifndef DG_EXP_NOUNPACK
                    const uint32_t ta_col = trow_a + sa * C::ACOLS + h * 32;
                    if (2 * h + 1 < nchunk) ptx::tmem_st_32x32b_x32(ta_col, ah);
                    else ptx::tmem_st_32x32b_x16(ta_col, ah);   // a half part: only its 16 columns are read
#else
                    if (ah[0] == 0x12345u && ah[3] == 0x777u) f16tab[1] = ah[2];
#endif
                }
                ptx::tmem_st_wait();
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(full_a(sa));
                if (lane == 0 && quarter == 0) TS_EV(2, g);
            }
        }
        }   // general stages
    } else {
        // ---------------- epilogue (lane quarter = warp % 4, tile group = warp / 4)
        constexpr int EG = NEPI / 4, HALF = CS ? BN / EG : BN, NCH = HALF / 32;
        static_assert(NCH % 2 == 0, "epilogue loads 64 columns at a time");
        // 16-bit requant offsets per column pair (bias_axis 0): negA = bias - (thr0 - 1), checked
        // against int16 overflow of acc + negA; any failure sends every tile to the 32-bit path
        if (!ta.early_b) ptx::griddep_wait();   // (the bias may come from the previous kernel)
        if (ta.f16 && ta.f16_res == 1 && threadIdx.x - EPI_WARP0 * 32 < 16)   // residual pair table (smem)
            f16tab[TAB_PAIRS - 16 + threadIdx.x - EPI_WARP0 * 32] = ta.res_pair[threadIdx.x - EPI_WARP0 * 32];
        if (ta.f16 && ta.f16_tab) {
            uint32_t bad = 0;
            for (int i = threadIdx.x - EPI_WARP0 * 32; i < (int)(ta.nq >> 1); i += NEPI * 32) {
                const int64_t n0 = (rq.bias ? (int64_t)__ldg(rq.bias + 2 * i) : 0) - ta.f16_thr0m1;
                const int64_t n1 = (rq.bias ? (int64_t)__ldg(rq.bias + 2 * i + 1) : 0) - ta.f16_thr0m1;
                if ((n0 < 0 ? -n0 : n0) + ta.f16_accmax > 32767 || (n1 < 0 ? -n1 : n1) + ta.f16_accmax > 32767) bad = 1;
                f16tab[i] = ((uint32_t)n0 & 0xFFFFu) | ((uint32_t)n1 << 16);
                if (ASM && ta.offs) {   // offset MMA operand rows 2i, 2i+1: n = 127 q + r, |r| <= 63
                    const int32_t qa = (int32_t)((n0 + (n0 >= 0 ? 63 : -63)) / 127), qb = (int32_t)((n1 + (n1 >= 0 ? 63 : -63)) / 127);
                    const int32_t ra = (int32_t)n0 - 127 * qa, rb = (int32_t)n1 - 127 * qb;
                    if (qa < -127 || qa > 127 || qb < -127 || qb > 127) *offs_bad = 1u;
                    const int c = 2 * i % BN, tb = 2 * i / BN;
                    uint8_t *blk = smem + C::OFF_OFFS + tb * BN * 32;
                    *reinterpret_cast<uint4 *>(blk + c * 16) = make_uint4((uint32_t)(qa & 0xFF) | ((uint32_t)(ra & 0xFF) << 8), 0, 0, 0);
                    *reinterpret_cast<uint4 *>(blk + (c + 1) * 16) = make_uint4((uint32_t)(qb & 0xFF) | ((uint32_t)(rb & 0xFF) << 8), 0, 0, 0);
                    *reinterpret_cast<uint4 *>(blk + BN * 16 + c * 16) = make_uint4(0, 0, 0, 0);
                    *reinterpret_cast<uint4 *>(blk + BN * 16 + (c + 1) * 16) = make_uint4(0, 0, 0, 0);
                }
            }
            if (bad) *f16_flag = 1u;
            if (ASM && ta.offs) {   // the constant A rows [127, 1, 0, ...] (second K chunk zero)
                uint8_t *one = smem + C::OFF_OFFS + 2 * BN * 32;
                for (int m = threadIdx.x - EPI_WARP0 * 32; m < BM; m += NEPI * 32) {
                    *reinterpret_cast<uint4 *>(one + m * 16) = make_uint4(0x17Fu, 0, 0, 0);
                    *reinterpret_cast<uint4 *>(one + BM * 16 + m * 16) = make_uint4(0, 0, 0, 0);
                }
                ptx::fence_proxy_async_smem();   // generic-proxy writes -> visible to the tensor core
            }
        }
        if (ta.f16 && (ta.f16_tab || ta.f16_res == 1)) ptx::named_bar_sync(EPI_BAR, NEPI * 32);
        if (ASM && ta.offs && lane == 0) ptx::mbar_arrive(sbase + C::OFF_OBAR);
        const bool f16_ok = ta.f16 && *f16_flag == 0u;
        const bool use_offs = ASM && ta.offs && f16_ok && *offs_bad == 0u;
        ptx::griddep_wait();
        if (!WIN && ((SK && ta.sk > 1) || ta.f16_res)) {
            epilogue_loop_rare<BN, NACC, EG, WIN, CS>(ta, rq, tmem, sbase + C::OFF_TAB, acc_full(0), ntiles, warp - EPI_WARP0,
                                                  lane, f16_ok);
        } else {
        const int quarter = warp & 3, eg = (warp - EPI_WARP0) >> 2, half = CS ? eg : 0;
        const bool col_bias = rq.bias && rq.bias_axis == 0;
        uint32_t tl = 0;
        const int wpair = WIN ? ta.wpair : 0;   // WIN pair mode: a work item = 2 row blocks (2 accumulators)
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
            if (!CS && EG > 1 && (int)(tl % EG) != eg) continue;
            int tp, tq;
            tile_coords(ta, t, tp, tq);
            for (int h = 0; h <= wpair; ++h) {
            const uint32_t u = (tl << wpair) + (uint32_t)h;   // accumulator use index
            const uint32_t acc = u % NACC;
            int64_t p = ((int64_t)tp << wpair) * BM + (int64_t)h * BM + quarter * 32 + lane;
            if (WIN) {   // padded pixel -> output pixel row, or np (not stored) for a padding position
                const int64_t q = p;
                p = ta.np;
                if (q < ta.nqv) {
                    const uint32_t b = fdiv((uint32_t)q, ta.fd_hpwp);
                    const uint32_t rem = (uint32_t)q - b * (uint32_t)((ta.H + 2) * ta.Wp);
                    const uint32_t hp = fdiv(rem, ta.fd_wp), wp = rem - hp * (uint32_t)ta.Wp;
                    if (hp >= 1 && hp <= (uint32_t)ta.H && wp >= 1 && wp <= (uint32_t)ta.W)
                        p = ((int64_t)b * ta.H + hp - 1) * ta.W + wp - 1;
                }
            }
            const int64_t q0 = (int64_t)tq * BN + half * HALF;
            if (lane == 0 && quarter == 0) TS_EV(8, tl);
            ptx::mbar_wait(acc_full(acc), (u / NACC) & 1u);
            if (lane == 0 && quarter == 0) TS_EV(9, tl);
            ptx::tc_fence_after();
            const uint32_t trow = tmem + acc * BN + half * HALF + ((uint32_t)(quarter * 32) << 16);
            const bool fast = ta.fast_rq && q0 + HALF <= ta.nq;
            const int32_t rb = (fast && rq.bias && rq.bias_axis == 1 && p < ta.np) ? __ldg(rq.bias + p) : 0;
            // 16-bit SIMD path (warp-uniform): per-row offsets need every lane's row in range
            bool use16 = fast && f16_ok;
#ifdef DG_EXP_NOEPI
            {
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(acc_empty(acc));
                continue;
            }
#endif
            uint32_t na_row = ta.f16_na2;
            if (use16 && !ta.f16_tab && rq.bias && rq.bias_axis == 1) {
                const int64_t n = (int64_t)rb - ta.f16_thr0m1;
                na_row = ((uint32_t)n & 0xFFFFu) * 0x10001u;
                use16 = __all_sync(0xFFFFFFFFu, (n < 0 ? -n : n) + ta.f16_accmax <= 32767);
            }
            if (use16) {
                if (ta.f16_tab && !use_offs) epi16_tile<HALF, 0, true>(ta, rq, trow, p, q0, na_row, sbase + C::OFF_TAB, lane, acc_empty(acc), tl);
                else epi16_tile<HALF, 0, false>(ta, rq, trow, p, q0, use_offs ? 0u : na_row, sbase + C::OFF_TAB, lane, acc_empty(acc), tl);
            } else if (C::STG_BYTES > 0 && ta.tma_d && !ta.has_rq && q0 + HALF <= ta.nq) {
                // int32 tile through the TMA tensor store: per 32-column chunk the warp's 32 rows x
                // 128 bytes go to its staging buffer (128-byte swizzle: 16-byte unit u of row r at
                // u ^ (r & 7), conflict-free STS.128) and one bulk tensor store writes them out; the
                // scattered per-lane row stores cost a wavefront per row (measured 21k cycles per
                // 128 x 256 int32 tile on the 16384^3 GEMM, with the single accumulator idle)
                const uint32_t stg = sbase + (uint32_t)C::OFF_STG + (uint32_t)(quarter * 4096);
                const int32_t row0 = (int32_t)(((int64_t)tp << wpair) * BM + quarter * 32);
#pragma unroll 1
                for (int c = 0; c < NCH; ++c) {
                    uint32_t v[32];
                    ptx::tmem_ld_32x32b_x32(trow + c * 32, v);
                    ptx::tmem_ld_wait();
                    if (c == NCH - 1) {
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(acc_empty(acc));
                    }
                    if (lane == 0) ptx::bulk_wait_read<0>();   // the previous chunk's store has read the buffer
                    __syncwarp();
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(stg + (uint32_t)lane * 128u +
                                                                                   ((uint32_t)(u ^ (lane & 7)) << 4)),
                                     "r"(v[4 * u]), "r"(v[4 * u + 1]), "r"(v[4 * u + 2]), "r"(v[4 * u + 3]) : "memory");
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        ptx::tma_store_2d(&tm_d, stg, (int32_t)(q0 + c * 32), row0);
                        for (int d = 0; d < ta.npeer; ++d) ptx::tma_store_2d(&pm.m[d], stg, (int32_t)(q0 + c * 32), row0);
                        ptx::bulk_commit();
                    }
                }
            } else if (!fast) {
#pragma unroll 1
                for (int c = 0; c < NCH; ++c) ts_epilogue_general(ta, rq, trow + c * 32, p, q0 + c * 32);
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(acc_empty(acc));
            } else {
                uint32_t r[32];
#pragma unroll 1
                for (int c = 0; c < NCH; ++c) {
                    const int64_t qc = q0 + c * 32;
                    int4 bx[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        bx[j] = col_bias ? __ldg(reinterpret_cast<const int4 *>(rq.bias + qc) + j) : make_int4(rb, rb, rb, rb);
                    ptx::tmem_ld_32x32b_x32(trow + c * 32, r);
                    ptx::tmem_ld_wait();
                    if (c == NCH - 1) {
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(acc_empty(acc));
                    }
                    if (p >= ta.np) continue;
                    // code = number of exact thresholds passed, from sign bits (|t|, |v| < 2^30)
                    uint32_t o0 = 0, o1 = 0;
                    if (ta.dir > 0) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int4 b4 = bx[j >> 2];
                            const int32_t b = (j & 3) == 0 ? b4.x : (j & 3) == 1 ? b4.y : (j & 3) == 2 ? b4.z : b4.w;
                            const int32_t v = (int32_t)r[j];
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
                            const int32_t v = (int32_t)r[j];
                            const uint32_t cd = ((uint32_t)(v + b - ta.thr[0] - 1) >> 31) + ((uint32_t)(v + b - ta.thr[1] - 1) >> 31) +
                                                ((uint32_t)(v + b - ta.thr[2] - 1) >> 31);
                            if (j < 16) o0 += cd << (2 * j);
                            else o1 += cd << (2 * (j - 16));
                        }
                    }
                    uint8_t *dp = reinterpret_cast<uint8_t *>(ta.D) + p * ta.ldd + (qc >> 2);
                    if ((reinterpret_cast<uintptr_t>(dp) & 7) == 0) *reinterpret_cast<uint2 *>(dp) = make_uint2(o0, o1);
                    else store_codes32_ts(dp, o0, o1, 8);
                }
            }
            if (lane == 0 && quarter == 0) TS_EV(10, tl);
            }   // h
        }
        }   // common modes
        if (C::STG_BYTES > 0 && ta.tma_d && lane == 0) ptx::bulk_wait<0>();   // TMA stores complete before exit
        if (ta.npeer) __threadfence_system();   // peer stores visible system-wide before the grid completes
    }

    ptx::tc_fence_before();
    __syncthreads();
#ifdef DG_TRACE
    if (blockIdx.x == 0)
        for (int i = threadIdx.x; i < TL_E * TL_N; i += blockDim.x) (&g_ts_tl[0][0])[i] = (&s_tl[0][0])[i];
#endif
    if (warp == PRODUCER_WARP) ptx::tmem_dealloc(tmem, C::TMEM_COLS);
    if (ta.bmc) ptx::cluster_sync_all();   // the partner's last multicast / commit into this CTA has landed
    if (SK && ta.sk > 1 && ta.sk_fused) {
        // every split's slice is stored (grid-wide barrier of the cooperative launch, with its memory
        // ordering): all threads of the grid sum the slices and requantise / store
        cooperative_groups::this_grid().sync();
        splitk_reduce_range(ta.ws_acc, ta.np, ta.nq, ta.sk, ta.D, ta.ldd, ta.has_rq, rq,
                            (int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
    }
}

// ---- Q expansion: packed codes -> int8 levels in the unpack16_levels order, zero beyond K.
// One thread per 16-byte packed chunk (64 codes -> 64 bytes).
__global__ void expand_operand_kernel(const uint8_t *__restrict__ packed, int64_t rows, int64_t K, int64_t ld,
                                      uint32_t L, int8_t *__restrict__ out, int64_t ld8) {
    const int64_t chunks = ld8 / 64;
    const int64_t total = rows * chunks;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / chunks, c = i - r * chunks;
        const int64_t k0 = c * 64;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (c * 16 + 16 <= ld) v = __ldg(reinterpret_cast<const uint4 *>(packed + r * ld + c * 16));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
        uint4 *dst = reinterpret_cast<uint4 *>(out + r * ld8 + k0);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint4 o = unpack16_levels(w[j], L);
            const int64_t kw = k0 + 16 * j;
            if (kw + 16 > K) {   // zero the bytes of codes >= K (no correction term needed)
                uint32_t ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
                for (int b = 0; b < 16; ++b) {
                    const int code = b < 8 ? 2 * b : 2 * (b - 8) + 1;   // inverse of the unpack order
                    if (kw + code >= K) ow[b >> 2] &= ~(0xFFu << (8 * (b & 3)));
                }
                o = make_uint4(ow[0], ow[1], ow[2], ow[3]);
            }
            dst[j] = o;
        }
    }
}

// ---------------------------------------------------------------- host
// Device copies of 16 pad-code bytes per pad code, each followed by 16 zero bytes (the cp.async
// sources of out-of-image and beyond-K taps of the implicit gather).
__device__ __align__(16) uint8_t g_pad_src[4][32];

const uint8_t *pad_source(int pad_code) {
    static const uint8_t *base = nullptr;
    if (!base) {
        uint8_t h[4][32] = {};
        for (int c = 0; c < 4; ++c)
            for (int i = 0; i < 16; ++i) h[c][i] = (uint8_t)(c | (c << 2) | (c << 4) | (c << 6));
        if (cudaMemcpyToSymbol(g_pad_src, h, sizeof(h)) != cudaSuccess) return nullptr;
        void *p = nullptr;
        if (cudaGetSymbolAddress(&p, g_pad_src) != cudaSuccess) return nullptr;
        base = reinterpret_cast<const uint8_t *>(p);
    }
    return base + 32 * (pad_code & 3);
}
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn_ts() {
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

// 2-D uint8 map over [rows][ld] with a {box_bytes, box_rows} box and the 128-byte swizzle
#ifdef DG_TRACE
extern "C" __attribute__((visibility("default"))) int dg_debug_ts_timeline(long long *host, int reset) {
    if (reset) {
        static long long z[TL_E * TL_N];
        return cudaMemcpyToSymbol(g_ts_tl, z, sizeof(z)) == cudaSuccess ? 0 : -1;
    }
    return cudaMemcpyFromSymbol(host, g_ts_tl, sizeof(long long) * TL_E * TL_N) == cudaSuccess ? 0 : -1;
}
#endif

bool make_map_sw128(CUtensorMap *m, const void *base, int64_t ld, int64_t rows, int box_rows, int box_bytes) {
    // swizzle span = box row bytes (16: none, 32, 64, 128)
    const CUtensorMapSwizzle sw = box_bytes >= 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : box_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : box_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
    EncodeTiledFn fn = encode_fn_ts();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld};
    cuuint32_t box[2] = {(cuuint32_t)box_bytes, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// extra all-gather destinations of the current lut_gemm_ts call (set there, read by launch_ts)
thread_local int32_t *const *g_peers = nullptr;
thread_local int32_t g_npeers = 0;
thread_local bool g_b_prepared = false;   // the B operand / bias are caller-prepared set-up data

template <int BN, int NEPI, int NUNP, int KST, bool WIN = false, bool ASM = false, bool SK = false, int EM = 0>
dg_status launch_ts(const uint8_t *P, int64_t ldp, const int8_t *Q8, int64_t ld8, int64_t np, int64_t nq, int64_t K,
                    const int32_t pl[4], const int32_t ql[4], void *D, int64_t ldd, const RequantArgs *rq,
                    cudaStream_t st, const TsConv *cv, void *skws = nullptr, size_t skws_bytes = 0) {
    using C = TsCfg<BN, (EM & EM_CSPLIT) ? 1 : NEPI / 4, KST, WIN, ASM, (EM & EM_A6) != 0>;
    int64_t acc_bound = 0;   // K * max |pl[a] * ql[b]|
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
            const int64_t e = (int64_t)pl[a] * ql[b];
            acc_bound = (e < 0 ? -e : e) > acc_bound ? (e < 0 ? -e : e) : acc_bound;
        }
    acc_bound *= K;
    TsArgs ta{};
    ta.np = np;
    ta.nq = nq;
    ta.nstages = (int32_t)((K + KST - 1) / KST);
    const int64_t kmma = (K + 31) / 32 * 32;
    ta.last_ksteps = (int32_t)((kmma - (int64_t)(ta.nstages - 1) * KST) / 32);
    ta.ntp = (int32_t)((np + BM - 1) / BM);
    if (WIN) {   // direct 3x3 conv: tiles over the padded pixel space
        const int64_t Wp = cv->W + 2, Hp = cv->H + 2, B = np / ((int64_t)cv->H * cv->W);
        ta.win = 1;
        ta.Wp = (int32_t)Wp;
        ta.nqv = B * Hp * Wp;
        if (ta.nqv >= ((int64_t)1 << 31)) return DG_ERR_SHAPE;
        if (np * cv->Cb >= ((int64_t)1 << 32)) return DG_ERR_UNSUPPORTED;   // (32-bit window fetch offsets)
        ta.ntp = (int32_t)((ta.nqv + BM - 1) / BM);
        // pair mode (tile mode on 64-wide tiles: C = 64, Cout <= 64, K = 576, weights resident): one window feeds 2 row blocks, so the halo rows are filled once per 2 blocks
        ta.wpair = ((BN == 64 || BN == 128) && KST == 256 && cv->Cb == 16 && K == 576 && nq <= BN && opt(OPT_WPAIR)) ? 1 : 0;
        if (ta.wpair) ta.ntp = (ta.ntp + 1) / 2;
        ta.WR = ((BM << ta.wpair) + 2 * (int32_t)Wp + 2 + 7) / 8 * 8;   // multiple of 8: LBO a multiple of 128 B
        // one window row per unpack thread, or up to 3 for C = 64 / 2 for C = 128
        if (ta.WR > NUNP * 32 && !((cv->Cb == 16 && ta.WR <= 3 * NUNP * 32) || (cv->Cb == 32 && ta.WR <= 2 * NUNP * 32)))
            return DG_ERR_UNSUPPORTED;
        ta.lbo = ta.WR * 16;
        int lg = 0;
        while ((1 << lg) < 4 * cv->Cb) ++lg;
        ta.clog2 = lg;
        ta.wslot = (ta.WR * cv->Cb + 127) / 128 * 128;
        ta.wbytes = (cv->Cb / 4) * ta.lbo;
        // (one window when only one fits: its fill then waits for the previous tile's MMAs)
        ta.nwin = (2 * ta.wslot + 3 * ta.wbytes <= C::P_REGION && C::SA >= 3) ? 3
                  : (2 * ta.wslot + 2 * ta.wbytes <= C::P_REGION ? 2 : 1);
        if (2 * ta.wslot + ta.nwin * ta.wbytes > C::P_REGION || ta.nwin > C::SA) return DG_ERR_UNSUPPORTED;
        ta.fd_hpwp = make_fastdiv((uint32_t)(Hp * Wp));
        ta.fd_wp = make_fastdiv((uint32_t)Wp);
        const int C = 4 * cv->Cb, nk = (int)(K / 32);
        if (nk > 72) return DG_ERR_UNSUPPORTED;
        for (int j = 0; j < nk; ++j) {
            const int tap = (32 * j) / C, c0 = (32 * j) % C, r = tap / 3, s = tap % 3;
            ta.koff[j] = (uint16_t)(((c0 / 16) * ta.lbo + (r * (int)Wp + s) * 16) >> 4);
        }
    }
    ta.ntq = (int32_t)((nq + BN - 1) / BN);
    ta.group = ta.ntq <= 4 ? 1 : (ta.ntp < 16 ? ta.ntp : 16);   // 1 = column block fastest
    ta.last_grp = (ta.ntp - 1) / ta.group;
    ta.last_rows = ta.ntp - ta.last_grp * ta.group;
    ta.fd_pg = make_fastdiv((uint32_t)(ta.group * ta.ntq));
    ta.fd_grp = make_fastdiv((uint32_t)ta.group);
    ta.fd_last = make_fastdiv((uint32_t)ta.last_rows);
    // packed P slots: TMA box {pks bytes, 128 rows} with the 128-byte swizzle; narrow rows
    // (short K) get many slots so that enough HBM reads are in flight per SM
    ta.bulk = (!cv && ldp <= 64 && ((uintptr_t)P & 15) == 0) ? 1 : 0;
    ta.pks = ta.bulk ? (int32_t)ldp : PKS_MAX;
    ta.P = P;
    ta.ldp = ldp;
    ta.sp = C::P_REGION / (BM * ta.pks);
    if (ta.sp > SP_MAX) ta.sp = SP_MAX;
    ta.bres = ((int64_t)ta.ntq * ta.nstages <= C::SB && opt(OPT_BRES)) ? 1 : 0;
    // weights (and bias) read before griddepcontrol.wait only when the caller declared them set-up data
    ta.early_b = (g_b_prepared && opt(OPT_EARLY_WEIGHTS)) ? 1 : 0;
    ta.lp = pack_levels_i8(pl);
    ta.D = D;
    ta.ldd = ldd;
    ta.has_rq = rq ? 1 : 0;
    ta.npeer = 0;
    if (g_npeers > 0) {   // fused all-gather: int32 output only, 16-byte aligned like D
        if (rq || g_npeers > 7) return DG_ERR_UNSUPPORTED;
        ta.npeer = g_npeers;
        for (int i = 0; i < g_npeers; ++i) {
            if (!g_peers[i] || (((uintptr_t)g_peers[i] ^ (uintptr_t)D) & 15)) return DG_ERR_INVALID_ARG;
            ta.peer[i] = g_peers[i];
        }
    }
    const bool has_res = rq && (rq->res || rq->res_codes);
    int64_t res_bound = 0;   // max |residual| for the 16-bit range check (int32 residuals: checked per warp)
    if (rq && rq->res_codes)
        for (int c = 0; c < 4; ++c) {
            const int64_t v = (int64_t)rq->res_levels[c] * rq->res_mult;
            res_bound = (v < 0 ? -v : v) > res_bound ? (v < 0 ? -v : v) : res_bound;
        }
    if (rq && acc_bound < ((int64_t)1 << 29) &&
        (!rq->bias || rq->bias_axis == 1 || (((uintptr_t)rq->bias) & 15) == 0)) {
        ta.fast_rq = has_res ? 0 : 1;   // acc is exact (no correction term): acc + bias >= t <=> x > t - 1
        ta.dir = rq->dir;
        for (int j = 0; j < 3; ++j) {
            const int64_t t = rq->thr[j];
            int64_t u = (t == INT64_MAX || t == INT64_MIN) ? t : (rq->dir > 0 ? t - 1 : t);
            const int64_t LIM = (int64_t)1 << 30;
            ta.thr[j] = (int32_t)(u > LIM ? LIM : (u < -LIM ? -LIM : u));
        }
        // 16-bit SIMD requant: |acc| < 2^15 (tcgen05.ld pack::16b keeps the low halves), finite
        // increasing thresholds, an (m, c) pair found; offsets checked here (uniform), per row
        // (in the epilogue) or per column (smem table at kernel start).
        const int64_t *t = rq->thr;
        uint32_t m16 = 0, c16 = 0;
        const bool res_ok = !has_res ||
                            (rq->res_codes && !rq->res && res_bound <= 16383 && (rq->ld_res_codes & 7) == 0 &&
                             (((uintptr_t)rq->res_codes) & 7) == 0) ||
                            (rq->res && !rq->res_codes && (rq->ld_res & 3) == 0 && (((uintptr_t)rq->res) & 15) == 0);
        if (rq->res && !rq->res_codes) res_bound = 16384;   // int32 residuals: |r| < 2^14 checked per chunk
        if (rq->dir > 0 && acc_bound + res_bound <= 32767 && t[0] > -((int64_t)1 << 30) && t[2] < ((int64_t)1 << 30) &&
            res_ok && (nq >> 1) <= TAB_PAIRS - 16 && opt(OPT_F16) && f16_params(t[0], t[1], t[2], m16, c16)) {
            const int64_t thr0m1 = t[0] - 1;
            ta.f16_m = m16;
            ta.f16_c2 = c16 * 0x10001u;
            ta.f16_w2 = (uint32_t)(t[2] - t[0] + 1) * 0x10001u;
            ta.f16_thr0m1 = (int32_t)thr0m1;
            ta.f16_accmax = (int32_t)(acc_bound + res_bound);
            ta.f16 = 1;
            if (WIN) {   // (the out-of-line residual loop has no padded-window row map)
            } else if (rq->res_codes) {
                ta.f16_res = 1;
                for (int i = 0; i < 16; ++i) {
                    const int32_t r0 = rq->res_levels[i & 3] * rq->res_mult, r1 = rq->res_levels[i >> 2] * rq->res_mult;
                    ta.res_pair[i] = ((uint32_t)r0 & 0xFFFFu) | ((uint32_t)r1 << 16);
                }
            } else if (rq->res) {
                ta.f16_res = 2;
            }
            ta.f16_tab = (!rq->bias || rq->bias_axis == 0) ? 1 : 0;   // else: per-row offsets
        }
    }
    // per-column offsets in the accumulator (see TsArgs::offs): every tile takes the 16-bit path
    ta.offs = (ASM && rq && ta.f16 && ta.f16_tab && ta.fast_rq && !ta.f16_res && nq % BN == 0 && nq / BN <= 2 &&
               opt(OPT_OFFS))
                  ? 1 : 0;
    if (cv) {
        ta.implicit = WIN ? 0 : 1;
        ta.X = cv->x;
        ta.H = cv->H;
        ta.W = cv->W;
        int lg = 0;
        while ((1 << lg) < cv->Cb) ++lg;
        ta.Cb_log2 = lg;
        ta.kw = cv->kw;
        ta.kw_recip = (65536 + cv->kw - 1) / cv->kw;
        ta.stride = cv->stride;
        ta.pad = cv->pad;
        ta.Ho = cv->Ho;
        ta.Wo = cv->Wo;
        ta.kb = cv->kh * cv->kw * cv->Cb;
        ta.padsrc = pad_source(cv->pad_code);
        if (!ta.padsrc) return DG_ERR_CUDA;
        ta.fd_wo = make_fastdiv((uint32_t)cv->Wo);
        ta.fd_ho = make_fastdiv((uint32_t)cv->Ho);
        if (np >= ((int64_t)1 << 31)) return DG_ERR_SHAPE;
    }
    CUtensorMap mp, mb, md, mbh;
    memset(&mp, 0, sizeof(mp));
    memset(&md, 0, sizeof(md));
    memset(&mbh, 0, sizeof(mbh));
    ta.tma_d = 0;
    PeerMaps pmaps;
    memset(&pmaps, 0, sizeof(pmaps));
    if (C::STG_BYTES > 0 && !rq && ((uintptr_t)D & 15) == 0 && (ldd * 4) % 16 == 0 && nq >= 32 && opt(OPT_TMA_STORE)) {
        EncodeTiledFn fn = encode_fn_ts();
        cuuint64_t dims[2] = {(cuuint64_t)nq, (cuuint64_t)np};
        cuuint64_t strides[1] = {(cuuint64_t)(ldd * 4)};
        cuuint32_t box[2] = {32, 32}, estr[2] = {1, 1};
        auto enc = [&](CUtensorMap *m, void *base) {
            return fn && fn(m, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        };
        bool ok = enc(&md, D);
        for (int i = 0; i < ta.npeer && ok; ++i) ok = enc(&pmaps.m[i], ta.peer[i]);
        ta.tma_d = ok ? 1 : 0;
    }
    if (!cv && !ta.bulk && !make_map_sw128(&mp, P, ldp, np, BM, ta.pks)) return DG_ERR_CUDA;
    if (!make_map_sw128(&mb, Q8, ld8, nq, BN, 128)) return DG_ERR_CUDA;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(lut_gemm_ts_kernel<BN, NEPI, NUNP, KST, WIN, ASM, SK, EM>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::ALLOC) !=
            cudaSuccess)
            return DG_ERR_CUDA;
        attr_set = true;
    }
    // split-K when the output tiles cannot fill the GPU and K is long (workspace for the slices given)
    ta.sk = 1;
    const int64_t otiles = (int64_t)ta.ntp * ta.ntq;
    if (SK && !ta.bulk && skws && otiles * 2 <= num_sms() && ta.nstages >= 4) {
        int64_t sk = num_sms() / otiles;
        sk = sk < ta.nstages / 2 ? sk : ta.nstages / 2;
        sk = sk < 8 ? sk : 8;
        const size_t need = (size_t)(sk * np * nq * 4);
        if (sk >= 2 && need <= skws_bytes) {
            ta.sk = (int32_t)sk;
            ta.fd_sk = make_fastdiv((uint32_t)sk);
            ta.ws_acc = reinterpret_cast<int32_t *>(skws);
            ta.sk_fused = opt(OPT_SKFUSE) ? 1 : 0;
        }
    }
    RequantArgs dummy{};
    const int64_t ntiles = otiles * ta.sk;
    if (ntiles > INT32_MAX) return DG_ERR_SHAPE;
    ta.nwork = (int32_t)ntiles;
    int grid = (int)(ntiles < num_sms() ? ntiles : num_sms());
    // B multicast across CTA pairs (see TsArgs::bmc): streamed B, no split-K, and a tile walk that
    // gives both CTAs of a pair the same column block at every step
    ta.bmc = (!WIN && !ASM && !ta.bres && ta.sk == 1 && opt(OPT_BMC) && (grid & ~1) >= 2 && ta.ntp % 2 == 0 &&
              ta.group % 2 == 0 && ta.last_rows % 2 == 0 && ntiles % 2 == 0 && ta.npeer == 0)
                 ? 1 : 0;
    if (ta.bmc) {
        grid &= ~1;
        if (!make_map_sw128(&mbh, Q8, ld8, nq, BN / 2, 128)) return DG_ERR_CUDA;
    }
    const RequantArgs rqv = rq ? *rq : dummy;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)grid);
    lc.blockDim = dim3((unsigned)Roles<NEPI, NUNP, EM>::NT);
    lc.dynamicSmemBytes = C::ALLOC;
    lc.stream = st;
    cudaLaunchAttribute la[2];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = opt(OPT_PDL) ? 1 : 0;
    if (ta.sk_fused) {
        la[1].id = cudaLaunchAttributeCooperative;   // (grid <= one CTA per SM: always co-resident)
        la[1].val.cooperative = 1;
    } else {
        la[1].id = cudaLaunchAttributeClusterDimension;
        la[1].val.clusterDim.x = 2;
        la[1].val.clusterDim.y = 1;
        la[1].val.clusterDim.z = 1;
    }
    lc.attrs = la;
    lc.numAttrs = (ta.sk_fused || ta.bmc) ? 2 : 1;
    if (cudaLaunchKernelEx(&lc, lut_gemm_ts_kernel<BN, NEPI, NUNP, KST, WIN, ASM, SK, EM>, mp, mb, md, pmaps, ta, rqv, mbh) !=
        cudaSuccess)
        return DG_ERR_CUDA;
    if (ta.sk > 1 && !ta.sk_fused) {
        const int64_t thr = np * ((nq + 3) >> 2);
        int64_t blocks = (thr + 255) / 256;
        if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
        lc.gridDim = dim3((unsigned)blocks);
        lc.blockDim = dim3(256);
        lc.dynamicSmemBytes = 0;
        if (cudaLaunchKernelEx(&lc, splitk_reduce_kernel, (const int32_t *)ta.ws_acc, np, nq, ta.sk, D, ldd,
                               (int32_t)(rq != nullptr), rqv) != cudaSuccess)
            return DG_ERR_CUDA;
    }
    char tag[160];
    snprintf(tag, sizeof(tag), "ts bn=%d epi=%d unp=%d kst=%d%s%s%s em=%d nwin=%d wpair=%d sk=%d bres=%d f16=%d implicit=%d bulk=%d early=%d tmad=%d bmc=%d offs=%d",
             BN, NEPI, NUNP, KST, WIN ? " win" : "", ASM ? " asm" : "", SK ? (ta.sk_fused ? " skinst fused" : " skinst") : "", EM, ta.nwin, ta.wpair, ta.sk,
             ta.bres, ta.f16, ta.implicit, ta.bulk, ta.early_b, ta.tma_d, ta.bmc, ta.offs);
    set_last_kernel(tag);
    return launch_status(ta.sk > 1 && !ta.sk_fused ? 2 : 1);
}

}  // namespace

// 16-bit SIMD requant parameters.  With x = clamp(acc + bias - (t0 - 1), 0, W), W = t2 - t0 + 1,
// the exact code is [x >= 1] + [x >= t1 - t0 + 1] + [x >= W]; find integers m, c with
// floor((x*m + c) / 2^14) equal to it.  x*m + c is monotone in x, so matching at the threshold
// boundaries suffices; the result is re-verified for every x in [0, W].
bool f16_params(int64_t t0, int64_t t1, int64_t t2, uint32_t &m_out, uint32_t &c_out) {
    const int64_t W = t2 - t0 + 1, X2 = t1 - t0 + 1;
    if (W < 1 || W > 16383 || X2 < 1 || X2 > W) return false;
    auto code = [&](int64_t x) { return (int64_t)(x >= 1) + (int64_t)(x >= X2) + (int64_t)(x >= W); };
    const int64_t pts[7] = {0, 0, 1, X2 - 1, X2, W - 1, W};
    for (int64_t m = 1; m * W < 65536; ++m) {
        int64_t lo = 0, hi = 65535;
        for (int i = 0; i < 7; ++i) {
            const int64_t x = pts[i], k = code(x);
            lo = lo > k * 16384 - x * m ? lo : k * 16384 - x * m;
            hi = hi < (k + 1) * 16384 - 1 - x * m ? hi : (k + 1) * 16384 - 1 - x * m;
        }
        if (lo > hi) continue;
        bool ok = true;
        for (int64_t x = 0; x <= W && ok; ++x) ok = (x * m + lo) >> 14 == code(x) && x * m + lo < 65536;
        if (!ok) continue;
        m_out = (uint32_t)m;
        c_out = (uint32_t)lo;
        return true;
    }
    return false;
}

int64_t expand_ld(int64_t K) { return (K + KA - 1) / KA * KA; }

dg_status expand_operand(const uint8_t *packed, int64_t rows, int64_t K, int64_t ld, const int32_t levels[4],
                         int8_t *out, int64_t ld8, cudaStream_t st) {
    if (rows == 0) return DG_OK;
    const int64_t work = rows * (ld8 / 64);
    int64_t blocks = (work + 255) / 256;
    const int64_t cap = (int64_t)num_sms() * 8;
    if (blocks > cap) blocks = cap;
    expand_operand_kernel<<<(int)blocks, 256, 0, st>>>(packed, rows, K, ld, pack_levels_i8(levels), out, ld8);
    return launch_status();
}

dg_status lut_gemm_ts(const uint8_t *P, int64_t ldp, const int8_t *Q8, int64_t ld8, int64_t np, int64_t nq, int64_t K,
                      const int32_t pl[4], const int32_t ql[4], void *D, int64_t ldd, const RequantArgs *rq,
                      cudaStream_t st, const TsConv *cv, void *skws, size_t skws_bytes, int32_t *const *peers,
                      int32_t npeers, bool b_prepared) {
    if (np > ((int64_t)1 << 31) - 1 || nq > ((int64_t)1 << 31) - 1) return DG_ERR_SHAPE;
    g_peers = peers;
    g_npeers = peers ? npeers : 0;
    g_b_prepared = b_prepared;
    struct Reset { ~Reset() { g_peers = nullptr; g_npeers = 0; g_b_prepared = false; } } reset;
    // (every switch below is read per call: dg_set_option, include/dg.h)
    const int64_t o_win = opt(OPT_WIN);
    // direct 3x3 / stride 1 / pad 1 convs: shifted-window kernel, which unpacks each input pixel once
    // per tile instead of once per tap.  Default for C = 64 (the "tile mode": one hand-off and 18
    // MMAs per tile, 3x3 64 -> 64 at 56x56 b256: 88 -> 54 us) and C = 128 with Cout <= 128 (weights
    // resident); C = 128 / 256 otherwise only when forced (measured no faster than the implicit gather)
    const bool win_shape = cv && cv->kh == 3 && cv->kw == 3 && cv->stride == 1 && cv->pad == 1;
    const bool two_waves = win_shape && (np / ((int64_t)cv->H * cv->W)) * (cv->H + 2) * (cv->W + 2) / BM >= 2 * num_sms();
    if (win_shape && cv->Cb == 32 && nq <= 128 && K == 1152 && o_win >= 0 && opt(OPT_WIN128) && (two_waves || o_win > 0)) {
        const dg_status s = launch_ts<128, 4, 8, 128, true>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv);
        if (s != DG_ERR_UNSUPPORTED) return s;
    }
    if (win_shape && cv->Cb >= 16 && cv->Cb <= 64 && (cv->Cb & (cv->Cb - 1)) == 0 && o_win >= 0 &&
        (o_win > 0 || (cv->Cb == 16 && nq <= 128 && two_waves))) {
        const dg_status s = nq > 64 ? launch_ts<128, 4, 8, 256, true>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv)
                                    : launch_ts<64, 4, 8, 256, true>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv);
        if (s != DG_ERR_UNSUPPORTED) return s;
    }
    // short K (<= 256 codes): the epilogue dominates -> two epilogue groups (EG = 2).
    // Stages of 256 codes (8 MMAs per hand-off) except where K <= 128 or BN = 256 (whose 128-code
    // stages already carry 512 MMA cycles).
    const bool short_k = K <= 2 * KA;
    // split-K candidates (few output tiles, K of >= 4 stages, workspace given): the SK instances
    const bool sk_on = opt(OPT_SPLITK) != 0;
    auto few = [&](int64_t bn) {
        return skws && sk_on && !short_k && ((np + BM - 1) / BM) * ((nq + bn - 1) / bn) * 2 <= num_sms();
    };
    const bool k256 = K > KA && opt(OPT_KST) != 128;
    // short K, wide output: 128x256 tiles with the A operand in shared memory and two TMEM accumulators
    // (measured: narrower ASM tiles with 128-code stages lose to the TMEM-A kernel at K = 256)
    if (short_k && nq >= 256 && opt(OPT_ASM)) {
        const int64_t em = opt(OPT_EM);
        if (em == 1) return launch_ts<256, 8, 4, 128, false, true, false, EM_CSPLIT>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv);
        if (em == 2) return launch_ts<256, 8, 4, 128, false, true, false, EM_HIGH>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv);
        if (em == 3) return launch_ts<256, 8, 4, 128, false, true, false, EM_CSPLIT | EM_HIGH>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv);
        if (em == 4) return launch_ts<256, 8, 4, 128, false, true, false, EM_A6>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv);
        if (em == 5) return launch_ts<256, 8, 4, 128, false, true, false, EM_A6 | EM_CSPLIT>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv);
        return launch_ts<256, 8, 4, 128, false, true>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv);
    }
    // 128x256 tiles halve the shared-memory bytes of B per MAC (measured: 8192^3 1666 -> 2323
    // TOPS); their single TMEM accumulator buffer cannot overlap the epilogue with the next tile,
    // so they are used only when the K loop is long (>= 24 x 128 codes).
    // 128x256 tiles for K >= 512 (measured: ResNet-50 stage-3 3x3 46 -> 35 us, downsamples -10%)
    const int64_t bn256_k = opt(OPT_BN256_K);
    const int64_t tiles256 = ((np + BM - 1) / BM) * ((nq + 255) / 256);
    if (nq >= 256 && K >= bn256_k && (tiles256 >= num_sms() || K >= 24 * KA) && opt(OPT_BN256))
        return few(256) ? launch_ts<256, 4, 8, 128, false, false, true>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv, skws, skws_bytes)
               : opt(OPT_UNP) == 12 ? launch_ts<256, 4, 12, 128>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv)
               : opt(OPT_UNP) == 16 ? launch_ts<256, 4, 16, 128>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv)
                                    : launch_ts<256, 4, 8, 128>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv);

    if (nq > 64 && !(short_k && opt(OPT_BN64_SHORT))) {
        if (short_k && !k256) return launch_ts<128, 8, 4, 128>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv);
        if (short_k) return launch_ts<128, 8, 4, 256>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv);
        if (few(128))
            return !k256 ? launch_ts<128, 4, 8, 128, false, false, true>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv, skws, skws_bytes)
                         : launch_ts<128, 4, 8, 256, false, false, true>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv, skws, skws_bytes);
        if (!k256) return launch_ts<128, 4, 8, 128>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv);
        return launch_ts<128, 4, 8, 256>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv);
    }
    if (short_k && !k256) return launch_ts<64, 8, 8, 128>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv);
    if (short_k) return launch_ts<64, 8, 8, 256>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv);
    if (few(64))
        return !k256 ? launch_ts<64, 4, 8, 128, false, false, true>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv, skws, skws_bytes)
                     : launch_ts<64, 4, 8, 256, false, false, true>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv, skws, skws_bytes);
    if (!k256) return launch_ts<64, 4, 8, 128>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv);
    return launch_ts<64, 4, 8, 256>(P, ldp, Q8, ld8, np, nq, K, pl, ql, D, ldd, rq, st, cv);
}

}  // namespace dg
