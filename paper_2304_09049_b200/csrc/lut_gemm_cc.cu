// lut_gemm_cc.cu — S5/S6/S7: the CUDA-core LUT-16 GEMM (the paper's method, Alg. 1
// P:221-242, mapped onto sm_100a integer pipes), valid for ANY 16-entry table.
//
//   D[p][q] = sum_{k<K} Tt[(P[p][k] << 2) | Q[q][k]]          (int32, exact)
//
// P and Q are packed 2-bit operands, K-major (dg.h).  The caller orients the table:
// Tt = T when P is the weight operand, Tt = T transposed when P is the activation side.
//
// Lookup mechanism (replaces AVX2 vpshufb):
//  * index nibbles (p<<2)|q for 16 code pairs of a 32-bit word pair are built with two
//    LOP3 per 8 nibbles from per-operand precomputed masks (the paper's unpack, Alg. 1 l.9);
//  * PRMT (byte permute) looks up 4 nibbles at once in an 8-byte half table held in two
//    registers.  The 16-entry table is split in a lo half (entries 0-7) and a hi half
//    (8-15); PRMT's sign-replicate bit (selector bit 3) returns 0x00 for the "wrong" half
//    because every stored byte is < 128 (entries are offset to be non-negative and split
//    into 6-bit chunks), so lo + hi is exactly the looked-up byte;
//  * byte lanes accumulate up to F words before a flush with IDP4A into int32
//    (the paper's 8-bit lane sums + horizontal reduce, made overflow-free).
// Exactness: the offset and the K padding (codes beyond K are 0 on both operands, dg.h)
// are removed with one exact integer correction per output.
#include "common.cuh"

namespace dg {

constexpr int kMaxChunks = 4;

struct CcTable {
    uint32_t t[kMaxChunks][4];  // per chunk: bytes 0-7 = lo half, 8-15 = hi half
    int32_t nch;
};

namespace {

constexpr int BP = 64, BQ = 64, KC_BYTES = 32, KC_WORDS = KC_BYTES / 4, SROW = 68;

DG_DEV uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

template <int NCH, int F>
__global__ void __launch_bounds__(256) lut_gemm_cc_kernel(
    const uint8_t *__restrict__ P, int64_t ldp, const uint8_t *__restrict__ Q, int64_t ldq,
    int64_t np, int64_t nq, int64_t nchunks, CcTable tab, int64_t corr, void *__restrict__ D,
    int64_t ldd, const __grid_constant__ RequantArgs rq, int has_rq) {
    __shared__ __align__(16) uint32_t Ps[2][KC_WORDS][SROW];
    __shared__ __align__(16) uint32_t Qs[2][KC_WORDS][SROW];

    const int tid = threadIdx.x;
    const int tq = tid & 15, tp = tid >> 4;
    const int64_t p0 = (int64_t)blockIdx.x * BP, q0 = (int64_t)blockIdx.y * BQ;

    // global->smem assignment: threads 0..127 load P, 128..255 load Q; 2 x 16 B per row
    const int ld_op = tid >> 7, ld_u = tid & 127, ld_h = ld_u & 1, ld_row = ld_u >> 1;
    const uint8_t *src_base;
    int64_t src_ld, src_rows, src_row;
    if (ld_op == 0) { src_base = P; src_ld = ldp; src_rows = np; src_row = p0 + ld_row; }
    else            { src_base = Q; src_ld = ldq; src_rows = nq; src_row = q0 + ld_row; }
    const bool row_ok = src_row < src_rows;
    const uint8_t *src_ptr = src_base + (row_ok ? src_row : 0) * src_ld + ld_h * 16;

    auto gload = [&](int64_t c) -> uint4 {
        const int64_t off = c * KC_BYTES;
        if (row_ok && off + ld_h * 16 < src_ld)
            return __ldg(reinterpret_cast<const uint4 *>(src_ptr + off));
        return make_uint4(0, 0, 0, 0);
    };
    auto sstore = [&](int buf, uint4 v) {
        uint32_t(*S)[SROW] = ld_op == 0 ? Ps[buf] : Qs[buf];
        S[4 * ld_h + 0][ld_row] = v.x;
        S[4 * ld_h + 1][ld_row] = v.y;
        S[4 * ld_h + 2][ld_row] = v.z;
        S[4 * ld_h + 3][ld_row] = v.w;
    };

    uint32_t t[NCH][4];
#pragma unroll
    for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int j = 0; j < 4; ++j) t[c][j] = tab.t[c][j];

    uint32_t acc[NCH][4][4];
    uint32_t accb[NCH][4][4];
#pragma unroll
    for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) { acc[c][i][j] = 0; accb[c][i][j] = 0; }

    uint4 pre = gload(0);
    sstore(0, pre);
    __syncthreads();

    for (int64_t ch = 0; ch < nchunks; ++ch) {
        const int buf = (int)(ch & 1);
        if (ch + 1 < nchunks) pre = gload(ch + 1);

#pragma unroll
        for (int w = 0; w < KC_WORDS; ++w) {
            const uint4 pw4 = *reinterpret_cast<const uint4 *>(&Ps[buf][w][tp * 4]);
            const uint4 qw4 = *reinterpret_cast<const uint4 *>(&Qs[buf][w][tq * 4]);
            const uint32_t pw[4] = {pw4.x, pw4.y, pw4.z, pw4.w};
            const uint32_t qw[4] = {qw4.x, qw4.y, qw4.z, qw4.w};
            uint32_t pa[4], pb[4], pa16[4], pb16[4], qa[4], qb[4], qa16[4], qb16[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                pa[i] = (pw[i] << 2) & 0xCCCCCCCCu;   // p codes 0,2,..,14 -> nibble bits 2-3
                pb[i] = pw[i] & 0xCCCCCCCCu;          // p codes 1,3,..,15
                pa16[i] = pa[i] >> 16;
                pb16[i] = pb[i] >> 16;
                qa[i] = qw[i] & 0x33333333u;          // q codes 0,2,..,14 -> nibble bits 0-1
                qb[i] = (qw[i] >> 2) & 0x33333333u;   // q codes 1,3,..,15
                qa16[i] = qa[i] >> 16;
                qb16[i] = qb[i] >> 16;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t s[4] = {pa[i] | qa[j], pa16[i] | qa16[j], pb[i] | qb[j],
                                           pb16[i] | qb16[j]};
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        const uint32_t sx = s[g] ^ 0x88888888u;
#pragma unroll
                        for (int c = 0; c < NCH; ++c) {
                            const uint32_t lo = prmt(t[c][0], t[c][1], s[g]);
                            const uint32_t hi = prmt(t[c][2], t[c][3], sx);
                            accb[c][i][j] += lo + hi;
                        }
                    }
                }
            if ((w + 1) % F == 0) {
#pragma unroll
                for (int c = 0; c < NCH; ++c)
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            acc[c][i][j] = __dp4a(accb[c][i][j], 0x01010101u, acc[c][i][j]);
                            accb[c][i][j] = 0;
                        }
            }
        }
        if (ch + 1 < nchunks) sstore(buf ^ 1, pre);
        __syncthreads();
    }

    // ---- epilogue: exact int32 result, optional fused requant (S7)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t p = p0 + tp * 4 + i;
        if (p >= np) continue;
        const int64_t qb0 = q0 + tq * 4;
        int32_t v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int64_t s = 0;
#pragma unroll
            for (int c = 0; c < NCH; ++c) s += (int64_t)acc[c][i][j] << (6 * c);
            v[j] = (int32_t)(s - corr);
        }
        if (!has_rq) {
            int32_t *Dp = reinterpret_cast<int32_t *>(D) + p * ldd + qb0;
            if (qb0 + 3 < nq && ((ldd & 3) == 0) && ((reinterpret_cast<uintptr_t>(D) & 15) == 0)) {
                *reinterpret_cast<int4 *>(Dp) = make_int4(v[0], v[1], v[2], v[3]);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (qb0 + j < nq) Dp[j] = v[j];
            }
        } else if (qb0 < nq) {
            uint32_t o = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (qb0 + j < nq) o |= requant_one(rq, v[j], p, qb0 + j) << (2 * j);
            reinterpret_cast<uint8_t *>(D)[p * ldd + (qb0 >> 2)] = (uint8_t)o;
        }
    }
}

}  // namespace

dg_status lut_gemm_cc(const uint8_t *P, int64_t ldp, const uint8_t *Q, int64_t ldq, int64_t np,
                      int64_t nq, int64_t K, const int32_t Tt[16], void *D, int64_t ldd,
                      const RequantArgs *rq, cudaStream_t st) {
    // offset the table to non-negative values and split it into 6-bit chunks
    int64_t mn = Tt[0], mx = Tt[0];
    for (int e = 1; e < 16; ++e) { mn = Tt[e] < mn ? Tt[e] : mn; mx = Tt[e] > mx ? Tt[e] : mx; }
    const int64_t off = -mn, range = mx - mn;
    int nch = 1;
    while (nch < kMaxChunks && (range >> (6 * nch)) != 0) ++nch;
    if ((range >> (6 * nch)) != 0) return DG_ERR_UNSUPPORTED;
    CcTable tab{};
    tab.nch = nch;
    for (int c = 0; c < nch; ++c)
        for (int e = 0; e < 16; ++e) {
            uint32_t b = (uint32_t)(((Tt[e] + off) >> (6 * c)) & 63);
            tab.t[c][e >> 2] |= b << (8 * (e & 3));
        }
    // each byte lane receives 4 chunk values (<= maxc) per word: flush before 255
    const int64_t maxc = nch == 1 ? range : 63;
    int64_t fw = maxc == 0 ? 8 : 255 / (4 * maxc);
    const int64_t nchunks = (K + 127) / 128;
    const int64_t Kp = nchunks * 128;
    const int64_t corr = off * Kp + (Kp - K) * (int64_t)Tt[0];
    RequantArgs dummy{};
    const RequantArgs &q = rq ? *rq : dummy;
    dim3 grid((unsigned)((np + BP - 1) / BP), (unsigned)((nq + BQ - 1) / BQ));
    if (grid.y > 65535) return DG_ERR_SHAPE;
    const int has = rq ? 1 : 0;
#define DG_CC_LAUNCH(NC, FW) \
    lut_gemm_cc_kernel<NC, FW><<<grid, 256, 0, st>>>(P, ldp, Q, ldq, np, nq, nchunks, tab, corr, D, ldd, q, has)
    if (nch == 1) {
        if (fw >= 8) DG_CC_LAUNCH(1, 8);
        else if (fw >= 4) DG_CC_LAUNCH(1, 4);
        else if (fw >= 2) DG_CC_LAUNCH(1, 2);
        else DG_CC_LAUNCH(1, 1);
    } else if (nch == 2) {
        DG_CC_LAUNCH(2, 1);
    } else if (nch == 3) {
        DG_CC_LAUNCH(3, 1);
    } else {
        DG_CC_LAUNCH(4, 1);
    }
#undef DG_CC_LAUNCH
    set_last_kernel(nch == 1 ? "cc nch=1" : nch == 2 ? "cc nch=2" : nch == 3 ? "cc nch=3" : "cc nch=4");
    return launch_status();
}

}  // namespace dg
