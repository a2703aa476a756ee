// api.cu — the C ABI of libdg (include/dg.h): host-side validation, LUT build (S4),
// variant dispatch and the conv orchestration (im2col + LUT GEMM + fused requant).
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

using namespace dg;

uint64_t &dg::launch_counter() {
    static uint64_t n = 0;
    return n;
}

namespace {

struct OptDesc {
    const char *name, *env;
    int64_t def;
    int64_t env_val;   // value an environment variable sets (its presence; DG_BN256_K: its number)
};
// name, initialising environment variable (ablation switches of DESIGN.md §6.1), default, env value
const OptDesc kOpts[dg::OPT_COUNT] = {
    {"win", "DG_WIN", 0, 1},            {"win128", "DG_NO_WIN128", 1, 0}, {"wpair", "DG_NO_WPAIR", 1, 0},
    {"asm", "DG_NO_ASM", 1, 0},         {"bn256", "DG_TS_NO_BN256", 1, 0}, {"bn256_k", "DG_BN256_K", 512, -1},
    {"kst", "DG_TS_K128", 0, 128},      {"bn64_short", "DG_BN64_SHORT", 0, 1}, {"splitk", "DG_NO_SPLITK", 1, 0},
    {"f16", "DG_NO_F16", 1, 0},         {"bres", "DG_NO_BRES", 1, 0},     {"pdl", "DG_NO_PDL", 1, 0},
    {"early_weights", "DG_EARLY_WEIGHTS", 0, 1}, {"f4conv", "DG_NO_F4CONV", 1, 0}, {"em", "DG_EM", 0, -1},
    {"tma_store", "DG_NO_TMA_STORE", 1, 0},      {"unp", "DG_UNP", 8, -1},
    {"f4_unp", "DG_F4_UNP", 0, -1},     {"f4_epi", "DG_F4_EPI", 0, -1},
    {"f4_bn", "DG_F4_BN", 0, -1},       {"f4_omma", "DG_F4_OMMA", 1, -1},
    {"f4_ct", "DG_F4_CT", 0, -1},       {"skfuse", "DG_SKFUSE", 0, 1},   {"f4_win", "DG_F4_WIN", 2, -1},
    {"offs", "DG_NO_OFFS", 1, 0},       {"bmc", "DG_BMC", 0, 1},         {"f4_wbres", "DG_F4_NO_WBRES", 1, 0},
    {"f4_i2c", "DG_F4_NO_I2C", 1, 0},   {"f4_w1x1", "DG_F4_W1X1", 1, 2},   {"f4_wpair", "DG_F4_NO_WPAIR", 1, 0},
};

int64_t *opt_table() {
    static int64_t v[dg::OPT_COUNT];
    static bool init = false;   // (first touch happens on the loading thread, before any call returns)
    if (!init) {
        for (int i = 0; i < dg::OPT_COUNT; ++i) {
            v[i] = kOpts[i].def;
            const char *e = getenv(kOpts[i].env);
            if (e) v[i] = kOpts[i].env_val >= 0 ? kOpts[i].env_val : atoll(e);
        }
        if (getenv("DG_NO_WIN")) v[dg::OPT_WIN] = -1;
        init = true;
    }
    return v;
}
__attribute__((constructor)) void opt_init() { opt_table(); }

thread_local char g_last_kernel[160] = "";

}  // namespace

int64_t dg::opt(dg::OptId id) { return __atomic_load_n(&opt_table()[id], __ATOMIC_RELAXED); }
void dg::set_last_kernel(const char *tag) {
    strncpy(g_last_kernel, tag, sizeof(g_last_kernel) - 1);
    g_last_kernel[sizeof(g_last_kernel) - 1] = 0;
}

namespace {

bool fits_bits(int64_t v, int32_t bits) {
    if (bits >= 32) return v >= INT32_MIN && v <= INT32_MAX;
    const int64_t lo = -((int64_t)1 << (bits - 1)), hi = ((int64_t)1 << (bits - 1)) - 1;
    return v >= lo && v <= hi;
}

bool aligned16(const void *p) { return ((uintptr_t)p & 15) == 0; }

int64_t max_abs_entry(const int32_t *e) {
    int64_t m = 0;
    for (int i = 0; i < 16; ++i) {
        int64_t a = e[i] < 0 ? -(int64_t)e[i] : e[i];
        m = a > m ? a : m;
    }
    return m;
}

bool levels_fit_i8(const int32_t *l) {
    for (int i = 0; i < 4; ++i)
        if (l[i] < -128 || l[i] > 127) return false;
    return true;
}

dg_status check_rq(const dg_requant *rq) {
    if (!rq) return DG_OK;
    if (rq->qmax < rq->qmin || rq->qmax - rq->qmin > 3 || rq->shift < 0 || rq->shift > 62)
        return DG_ERR_RANGE;
    if (rq->bias_axis != 0 && rq->bias_axis != 1) return DG_ERR_INVALID_ARG;
    if (rq->d_res_codes)
        for (int i = 0; i < 4; ++i) {
            const int64_t r = (int64_t)rq->res_levels[i] * rq->res_mult;
            if (r > INT32_MAX || r < INT32_MIN) return DG_ERR_RANGE;   // keeps |v| < 2^34
        }
    return DG_OK;
}

// D[p][q] = sum_k Tt[(P<<2)|Q]; pl/ql = per-code levels of P/Q (valid iff product).
// variant 2 (tc) expands Q into the workspace, then runs the TMEM-A kernel.
dg_status gemm_dispatch(const uint8_t *P, int64_t ldp, const uint8_t *Q, int64_t ldq, int64_t np,
                        int64_t nq, int64_t K, const int32_t Tt[16], bool is_product,
                        const int32_t pl[4], const int32_t ql[4], void *D, int64_t ldd,
                        const dg_requant *rq, void *ws, size_t ws_bytes, int32_t variant, cudaStream_t st) {
    RequantArgs a{};
    const RequantArgs *ap = nullptr;
    if (rq) { a = to_args(rq); ap = &a; }
    const bool tc_ok = is_product && levels_fit_i8(pl) && levels_fit_i8(ql) && tc_available();
    // non-product table with int8 entries: the one-hot K' = 4K form on the tensor cores (dg.h)
    const bool oh_ok = !is_product && max_abs_entry(Tt) <= 127 && tc_available() && (ldp % 4) == 0 &&
                       (((uintptr_t)P) & 3) == 0;
    if (variant == 3 && !tc_ok) return DG_ERR_UNSUPPORTED;
    if (variant == 2 && !tc_ok && !oh_ok) return DG_ERR_UNSUPPORTED;
    if ((variant == 0 || variant == 2) && !tc_ok && oh_ok) {
        // P' = one-hot(P) [np][onehot_ld(K)], Q' = table columns of Q [nq][tcols_ld(K)]:
        // D[p][q] = sum_k sum_i [P[p][k] == i] * Tt[(i << 2) | Q[q][k]]
        const int64_t l1 = onehot_ld(K), lt = tcols_ld(K);
        uint8_t *p1 = (uint8_t *)(((uintptr_t)ws + 127) & ~(uintptr_t)127);
        int8_t *qt = (int8_t *)(((uintptr_t)(p1 + np * l1) + 127) & ~(uintptr_t)127);
        if (!ws || (uint8_t *)(qt + nq * lt) > (uint8_t *)ws + ws_bytes) return DG_ERR_WORKSPACE;
        dg_status s = expand_onehot(P, np, K, ldp, p1, l1, st);
        if (s != DG_OK) return s;
        s = expand_tcols(Q, nq, K, ldq, Tt, qt, lt, st);
        if (s != DG_OK) return s;
        const int32_t emax = (int32_t)max_abs_entry(Tt);
        const int32_t pl1[4] = {0, 1, 0, 0}, ql1[4] = {emax, 0, 0, 0};   // (ql1 only bounds |acc|)
        return lut_gemm_ts(p1, l1, qt, lt, np, nq, 4 * K, pl1, ql1, D, ldd, ap, st);
    }
    if (variant == 3) return lut_gemm_tc(P, ldp, Q, ldq, np, nq, K, pl, ql, D, ldd, ap, st);
    if (variant == 2 || (variant == 0 && tc_ok)) {
        const int64_t ld8 = expand_ld(K);
        int8_t *q8 = (int8_t *)(((uintptr_t)ws + 127) & ~(uintptr_t)127);
        if (!ws || (int64_t)ws_bytes - (int64_t)((uint8_t *)q8 - (uint8_t *)ws) < nq * ld8) return DG_ERR_WORKSPACE;
        dg_status s = expand_operand(Q, nq, K, ldq, ql, q8, ld8, st);
        if (s != DG_OK) return s;
        return lut_gemm_ts(P, ldp, q8, ld8, np, nq, K, pl, ql, D, ldd, ap, st);
    }
    return lut_gemm_cc(P, ldp, Q, ldq, np, nq, K, Tt, D, ldd, ap, st);
}

}  // namespace

extern "C" {

const char *dg_status_string(dg_status s) {
    switch (s) {
        case DG_OK: return "DG_OK";
        case DG_ERR_INVALID_ARG: return "DG_ERR_INVALID_ARG";
        case DG_ERR_SHAPE: return "DG_ERR_SHAPE";
        case DG_ERR_RANGE: return "DG_ERR_RANGE";
        case DG_ERR_OVERFLOW: return "DG_ERR_OVERFLOW";
        case DG_ERR_UNSUPPORTED: return "DG_ERR_UNSUPPORTED";
        case DG_ERR_CUDA: return "DG_ERR_CUDA";
        case DG_ERR_WORKSPACE: return "DG_ERR_WORKSPACE";
        default: return "DG_ERR_UNKNOWN";
    }
}

int32_t dg_abi_version(void) { return DG_ABI_VERSION; }

uint64_t dg_kernel_launches(void) { return __atomic_load_n(&dg::launch_counter(), __ATOMIC_RELAXED); }

dg_status dg_set_option(const char *name, int64_t value) {
    if (!name) return DG_ERR_INVALID_ARG;
    for (int i = 0; i < dg::OPT_COUNT; ++i)
        if (!strcmp(name, kOpts[i].name)) {
            __atomic_store_n(&opt_table()[i], value, __ATOMIC_RELAXED);
            return DG_OK;
        }
    return DG_ERR_INVALID_ARG;
}

dg_status dg_get_option(const char *name, int64_t *value) {
    if (!name || !value) return DG_ERR_INVALID_ARG;
    for (int i = 0; i < dg::OPT_COUNT; ++i)
        if (!strcmp(name, kOpts[i].name)) {
            *value = dg::opt((dg::OptId)i);
            return DG_OK;
        }
    return DG_ERR_INVALID_ARG;
}

dg_status dg_reset_options(void) {
    for (int i = 0; i < dg::OPT_COUNT; ++i) __atomic_store_n(&opt_table()[i], kOpts[i].def, __ATOMIC_RELAXED);
    return DG_OK;
}

const char *dg_last_kernel(void) { return g_last_kernel; }

dg_status dg_build_lut(const int32_t wl[4], const int32_t al[4], int32_t entry_bits, dg_lut *out) {
    if (!wl || !al || !out) return DG_ERR_INVALID_ARG;
    if (entry_bits != 8 && entry_bits != 16 && entry_bits != 32) return DG_ERR_INVALID_ARG;
    dg_lut t;
    memset(&t, 0, sizeof(t));
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            const int64_t v = (int64_t)wl[i] * al[j];  // LUT-16 entry: w·a
            if (!fits_bits(v, entry_bits)) return DG_ERR_OVERFLOW;
            t.entries[(i << 2) | j] = (int32_t)v;
        }
    t.entry_bits = entry_bits;
    t.is_product = 1;
    for (int i = 0; i < 4; ++i) { t.wl[i] = wl[i]; t.al[i] = al[i]; }
    *out = t;
    return DG_OK;
}

dg_status dg_lut_from_table(const int32_t entries[16], int32_t entry_bits, dg_lut *out) {
    if (!entries || !out) return DG_ERR_INVALID_ARG;
    if (entry_bits != 8 && entry_bits != 16 && entry_bits != 32) return DG_ERR_INVALID_ARG;
    dg_lut t;
    memset(&t, 0, sizeof(t));
    for (int e = 0; e < 16; ++e) {
        if (!fits_bits(entries[e], entry_bits)) return DG_ERR_OVERFLOW;
        t.entries[e] = entries[e];
    }
    t.entry_bits = entry_bits;
    t.is_product = 0;
    *out = t;
    return DG_OK;
}

size_t dg_lut_gemm_workspace_size(int64_t M, int64_t N, int64_t K) {
    if (M <= 0 || N <= 0 || K <= 0) return 0;
    const int64_t product = N * expand_ld(K) + 128;
    const int64_t onehot = M * onehot_ld(K) + 128 + N * tcols_ld(K) + 128;   // non-product int8 tables
    return (size_t)(product > onehot ? product : onehot);
}

dg_status dg_lut_gemm(const uint8_t *d_w, int64_t ldw, const uint8_t *d_at, int64_t lda, int64_t M,
                      int64_t N, int64_t K, const dg_lut *lut, void *d_c, int64_t ldc,
                      const dg_requant *rq, void *d_ws, size_t ws_bytes, int32_t variant, void *stream) {
    if (!d_w || !d_at || !lut || !d_c) return DG_ERR_INVALID_ARG;
    if (variant < 0 || variant > 3) return DG_ERR_INVALID_ARG;
    if (M <= 0 || N <= 0 || K <= 0) return DG_ERR_SHAPE;
    if (ldw % 16 || lda % 16 || ldw * 4 < K || lda * 4 < K) return DG_ERR_SHAPE;
    if (!aligned16(d_w) || !aligned16(d_at)) return DG_ERR_INVALID_ARG;
    if (rq ? (ldc * 4 < N) : (ldc < N)) return DG_ERR_SHAPE;
    dg_status s = check_rq(rq);
    if (s != DG_OK) return s;
    if ((int64_t)K * max_abs_entry(lut->entries) >= ((int64_t)1 << 31)) return DG_ERR_OVERFLOW;
    // P = W (rows m), Q = At (rows n): D[m][n] = C[m][n], table index (w<<2)|a as is.
    return gemm_dispatch(d_w, ldw, d_at, lda, M, N, K, lut->entries, lut->is_product != 0, lut->wl,
                         lut->al, d_c, ldc, rq, d_ws, ws_bytes, variant, (cudaStream_t)stream);
}

int64_t dg_expand_ld(int64_t K) { return K <= 0 ? 0 : expand_ld(K); }

dg_status dg_expand_operand(const uint8_t *d_packed, int64_t rows, int64_t K, int64_t ld,
                            const int32_t levels[4], int8_t *d_out, int64_t ld_out, void *stream) {
    if (!d_packed || !levels || !d_out) return DG_ERR_INVALID_ARG;
    if (rows < 0 || K <= 0 || ld % 16 || ld * 4 < K || ld_out < expand_ld(K) || ld_out % 128) return DG_ERR_SHAPE;
    if (!levels_fit_i8(levels)) return DG_ERR_RANGE;
    if (!aligned16(d_packed) || ((uintptr_t)d_out & 127)) return DG_ERR_INVALID_ARG;
    return expand_operand(d_packed, rows, K, ld, levels, d_out, ld_out, (cudaStream_t)stream);
}

int64_t dg_onehot_ld(int64_t K) { return K <= 0 ? 0 : onehot_ld(K); }
int64_t dg_tcols_ld(int64_t K) { return K <= 0 ? 0 : tcols_ld(K); }

dg_status dg_expand_onehot(const uint8_t *d_w, int64_t rows, int64_t K, int64_t ld, uint8_t *d_out, int64_t ld_out,
                           void *stream) {
    if (!d_w || !d_out) return DG_ERR_INVALID_ARG;
    if (rows < 0 || K <= 0 || ld * 4 < K || ld % 4 || ld_out < onehot_ld(K) || ld_out % 16) return DG_ERR_SHAPE;
    if (((uintptr_t)d_w & 3) || !aligned16(d_out)) return DG_ERR_INVALID_ARG;
    return expand_onehot(d_w, rows, K, ld, d_out, ld_out, (cudaStream_t)stream);
}

dg_status dg_expand_tcols(const uint8_t *d_at, int64_t rows, int64_t K, int64_t ld, const dg_lut *lut, int8_t *d_out,
                          int64_t ld_out, void *stream) {
    if (!d_at || !lut || !d_out) return DG_ERR_INVALID_ARG;
    if (rows < 0 || K <= 0 || ld * 4 < K || ld_out < tcols_ld(K) || ld_out % 128) return DG_ERR_SHAPE;
    if ((uintptr_t)d_out & 127) return DG_ERR_INVALID_ARG;
    if (max_abs_entry(lut->entries) > 127) return DG_ERR_UNSUPPORTED;
    return expand_tcols(d_at, rows, K, ld, lut->entries, d_out, ld_out, (cudaStream_t)stream);
}

dg_status dg_lut_gemm_onehot(const uint8_t *d_w1h, int64_t ldw1h, const int8_t *d_atc, int64_t ldatc, int64_t M,
                             int64_t N, int64_t K, const dg_lut *lut, void *d_c, int64_t ldc, const dg_requant *rq,
                             void *stream) {
    if (!d_w1h || !d_atc || !lut || !d_c) return DG_ERR_INVALID_ARG;
    if (M <= 0 || N <= 0 || K <= 0) return DG_ERR_SHAPE;
    if (ldw1h % 16 || ldw1h < onehot_ld(K) || ldatc < tcols_ld(K) || ldatc % 128) return DG_ERR_SHAPE;
    if (!aligned16(d_w1h) || ((uintptr_t)d_atc & 127)) return DG_ERR_INVALID_ARG;
    if (rq ? (ldc * 4 < N) : (ldc < N)) return DG_ERR_SHAPE;
    dg_status s = check_rq(rq);
    if (s != DG_OK) return s;
    const int64_t emax = max_abs_entry(lut->entries);
    if (emax > 127 || !tc_available()) return DG_ERR_UNSUPPORTED;
    if (K * emax >= ((int64_t)1 << 31)) return DG_ERR_OVERFLOW;
    RequantArgs a{};
    if (rq) a = to_args(rq);
    // one-hot side: codes 0 / 1 with identity levels; the expanded side's "levels" only bound |acc|
    const int32_t pl[4] = {0, 1, 0, 0}, ql[4] = {(int32_t)emax, 0, 0, 0};
    return lut_gemm_ts(d_w1h, ldw1h, d_atc, ldatc, M, N, 4 * K, pl, ql, d_c, ldc, rq ? &a : nullptr,
                       (cudaStream_t)stream, nullptr, nullptr, 0, nullptr, 0, true);
}

// ---- general 4-bit (and 3-bit) tables: one-hot over the 16 weight codes, K' = 16K (dg.h)
static int64_t max_abs256(const int32_t *t) {
    int64_t m = 0;
    for (int e = 0; e < 256; ++e) m = (t[e] < 0 ? -(int64_t)t[e] : t[e]) > m ? (t[e] < 0 ? -(int64_t)t[e] : t[e]) : m;
    return m;
}

int64_t dg_onehot4_ld(int64_t K) { return K <= 0 ? 0 : onehot4_ld(K); }
int64_t dg_tcols4_ld(int64_t K) { return K <= 0 ? 0 : tcols4_ld(K); }

dg_status dg_expand_onehot4(const uint8_t *d_w4, int64_t rows, int64_t K, int64_t ld, uint8_t *d_out, int64_t ld_out,
                            void *stream) {
    if (!d_w4 || !d_out) return DG_ERR_INVALID_ARG;
    if (rows < 0 || K <= 0 || ld * 2 < K || ld_out < onehot4_ld(K) || ld_out % 16) return DG_ERR_SHAPE;
    if (!aligned16(d_out)) return DG_ERR_INVALID_ARG;
    return expand_onehot4(d_w4, rows, K, ld, d_out, ld_out, (cudaStream_t)stream);
}

dg_status dg_expand_tcols4(const uint8_t *d_at4, int64_t rows, int64_t K, int64_t ld, const int32_t table[256],
                           int8_t *d_out, int64_t ld_out, void *stream) {
    if (!d_at4 || !table || !d_out) return DG_ERR_INVALID_ARG;
    if (rows < 0 || K <= 0 || ld * 2 < K || ld_out < tcols4_ld(K) || ld_out % 128) return DG_ERR_SHAPE;
    if ((uintptr_t)d_out & 127) return DG_ERR_INVALID_ARG;
    if (max_abs256(table) > 127) return DG_ERR_UNSUPPORTED;
    return expand_tcols4(d_at4, rows, K, ld, table, d_out, ld_out, (cudaStream_t)stream);
}

dg_status dg_lut_gemm4_onehot(const uint8_t *d_w1h, int64_t ldw1h, const int8_t *d_atc, int64_t ldatc, int64_t M, int64_t N,
                              int64_t K, const int32_t table[256], void *d_c, int64_t ldc, const dg_requant *rq,
                              void *stream) {
    if (!d_w1h || !d_atc || !table || !d_c) return DG_ERR_INVALID_ARG;
    if (M <= 0 || N <= 0 || K <= 0) return DG_ERR_SHAPE;
    if (ldw1h % 16 || ldw1h < onehot4_ld(K) || ldatc < tcols4_ld(K) || ldatc % 128) return DG_ERR_SHAPE;
    if (!aligned16(d_w1h) || ((uintptr_t)d_atc & 127)) return DG_ERR_INVALID_ARG;
    if (rq ? (ldc * 4 < N) : (ldc < N)) return DG_ERR_SHAPE;
    dg_status s = check_rq(rq);
    if (s != DG_OK) return s;
    const int64_t emax = max_abs256(table);
    if (emax > 127 || !tc_available()) return DG_ERR_UNSUPPORTED;
    if (K * emax >= ((int64_t)1 << 31)) return DG_ERR_OVERFLOW;
    RequantArgs a{};
    if (rq) a = to_args(rq);
    const int32_t pl[4] = {0, 1, 0, 0}, ql[4] = {(int32_t)emax, 0, 0, 0};   // (ql only bounds |acc|)
    return lut_gemm_ts(d_w1h, ldw1h, d_atc, ldatc, M, N, 16 * K, pl, ql, d_c, ldc, rq ? &a : nullptr,
                       (cudaStream_t)stream, nullptr, nullptr, 0, nullptr, 0, true);
}

// ---- 4-bit operands as 2-bit digit pairs (dg.h)
static int32_t max_abs16(const int32_t *l) {
    int32_t m = 0;
    for (int i = 0; i < 16; ++i) m = (l[i] < 0 ? -l[i] : l[i]) > m ? (l[i] < 0 ? -l[i] : l[i]) : m;
    return m;
}

dg_status dg_expand_digits4(const uint8_t *d_w4, int64_t rows, int64_t K, int64_t ld, const int32_t levels[16],
                            int8_t *d_out, int64_t ld_out, void *stream) {
    if (!d_w4 || !d_out || !levels) return DG_ERR_INVALID_ARG;
    if (rows < 0 || K <= 0 || ld * 2 < K || ld_out < expand_ld(2 * K) || ld_out % 128) return DG_ERR_SHAPE;
    if ((uintptr_t)d_out & 127) return DG_ERR_INVALID_ARG;
    if (4 * max_abs16(levels) > 127) return DG_ERR_RANGE;
    return expand_digits4(d_w4, rows, K, ld, levels, d_out, ld_out, (cudaStream_t)stream);
}

dg_status dg_lut_gemm4_prepared(const uint8_t *d_at4, int64_t lda, const int8_t *d_w8, int64_t ld8, int64_t N, int64_t M,
                                int64_t K, const int32_t levels[16], void *d_ct, int64_t ldct, const dg_requant *rq,
                                void *stream) {
    if (!d_at4 || !d_w8 || !levels || !d_ct) return DG_ERR_INVALID_ARG;
    if (M <= 0 || N <= 0 || K <= 0) return DG_ERR_SHAPE;
    if (lda % 16 || lda * 2 < K || ld8 < expand_ld(2 * K) || ld8 % 128) return DG_ERR_SHAPE;
    if (!aligned16(d_at4) || ((uintptr_t)d_w8 & 127)) return DG_ERR_INVALID_ARG;
    if (rq ? (ldct * 4 < M) : (ldct < M)) return DG_ERR_SHAPE;
    dg_status s = check_rq(rq);
    if (s != DG_OK) return s;
    const int32_t wmax = max_abs16(levels);
    if (4 * wmax > 127) return DG_ERR_RANGE;
    if (!tc_available()) return DG_ERR_UNSUPPORTED;
    if (K * 15 * (int64_t)wmax >= ((int64_t)1 << 31)) return DG_ERR_OVERFLOW;
    RequantArgs a{};
    if (rq) a = to_args(rq);
    // digit side: identity levels; the weights' side levels only bound |acc| (true bound 15 K wmax)
    const int32_t pl[4] = {0, 1, 2, 3}, ql[4] = {(5 * wmax + 1) / 2, 0, 0, 0};
    return lut_gemm_ts(d_at4, lda, d_w8, ld8, N, M, 2 * K, pl, ql, d_ct, ldct, rq ? &a : nullptr, (cudaStream_t)stream,
                       nullptr, nullptr, 0, nullptr, 0, true);
}

dg_status dg_float_table_fixed(const float table[16], int32_t digits[48], int32_t *shift) {
    if (!table || !digits || !shift) return DG_ERR_INVALID_ARG;
    for (int e = 0; e < 16; ++e)
        if (!isfinite(table[e])) return DG_ERR_RANGE;
    int32_t d[3][16];
    float_table_digits(table, d, shift);
    for (int j = 0; j < 3; ++j)
        for (int e = 0; e < 16; ++e) digits[16 * j + e] = d[j][e];
    return DG_OK;
}

size_t dg_lut_gemm_f32_workspace_size(int64_t M, int64_t N, int64_t K) {
    if (M <= 0 || N <= 0 || K <= 0) return 0;
    return (size_t)lut_gemm_f32_workspace(M, N, K);
}

dg_status dg_lut_gemm_f32(const uint8_t *d_w, int64_t ldw, const uint8_t *d_at, int64_t lda, int64_t M, int64_t N,
                          int64_t K, const float table[16], float *d_c, int64_t ldc, void *d_ws, size_t ws_bytes,
                          void *stream) {
    if (!d_w || !d_at || !table || !d_c || !d_ws) return DG_ERR_INVALID_ARG;
    if (M <= 0 || N <= 0 || K <= 0) return DG_ERR_SHAPE;
    if (ldw % 16 || lda % 16 || ldw * 4 < K || lda * 4 < K || ldc < N) return DG_ERR_SHAPE;
    if (!aligned16(d_w) || !aligned16(d_at)) return DG_ERR_INVALID_ARG;
    for (int e = 0; e < 16; ++e)
        if (!isfinite(table[e])) return DG_ERR_RANGE;
    if (K >= ((int64_t)1 << 22)) return DG_ERR_OVERFLOW;   // digit sums K * 4 * 128 < 2^31
    if (!tc_available()) return DG_ERR_UNSUPPORTED;
    if (ws_bytes < (size_t)lut_gemm_f32_workspace(M, N, K)) return DG_ERR_WORKSPACE;
    return lut_gemm_f32(d_w, ldw, d_at, lda, M, N, K, table, d_c, ldc, d_ws, ws_bytes, (cudaStream_t)stream);
}

dg_status dg_lut_conv2d_f4_prepared(const uint8_t *d_x, const uint8_t *d_w4, int64_t ld4, const dg_lut *lut,
                                    const dg_conv_params *p, const dg_requant *rq, void *d_out, void *stream) {
    if (!d_x || !d_w4 || !lut || !p || !d_out) return DG_ERR_INVALID_ARG;
    if (p->B <= 0 || p->H <= 0 || p->W <= 0 || p->C <= 0 || p->Cout <= 0 || p->kh <= 0 || p->kw <= 0 ||
        p->stride <= 0 || p->pad < 0)
        return DG_ERR_SHAPE;
    if (p->C % 4 || p->pad_code < 0 || p->pad_code > 3) return DG_ERR_RANGE;
    if (rq && p->Cout % 4) return DG_ERR_SHAPE;
    const int64_t Ho = (p->H + 2 * p->pad - p->kh) / p->stride + 1;
    const int64_t Wo = (p->W + 2 * p->pad - p->kw) / p->stride + 1;
    if (Ho <= 0 || Wo <= 0) return DG_ERR_SHAPE;
    const int64_t K = (int64_t)p->kh * p->kw * p->C;
    if (ld4 < expand_f4_ld(K) || ld4 % 128 || !aligned16(d_w4) || !aligned16(d_x)) return DG_ERR_SHAPE;
    dg_status s = check_rq(rq);
    if (s != DG_OK) return s;
    if (!lut->is_product || !tc_available()) return DG_ERR_UNSUPPORTED;
    for (int c = 0; c < 4; ++c)
        if (lut->al[c] != c || f4_nibble_half(lut->wl[c]) < 0) return DG_ERR_UNSUPPORTED;
    const int64_t acc_bound = K * max_abs_entry(lut->entries);
    if (acc_bound >= ((int64_t)1 << 22)) return DG_ERR_OVERFLOW;
    // the pad code's level must be exact in e2m1 too: codes are e2m1 already, nothing to check
    RequantArgs ra{};
    if (rq) ra = to_args(rq);
    TsConv cv{d_x, p->H, p->W, p->C / 4, p->kh, p->kw, p->stride, p->pad, (int32_t)Ho, (int32_t)Wo, p->pad_code};
    return lut_conv_f4(d_x, d_w4, ld4, cv, (int64_t)p->B * Ho * Wo, p->Cout, K, acc_bound, d_out,
                       rq ? p->Cout / 4 : p->Cout, rq ? &ra : nullptr, (cudaStream_t)stream, true);
}

dg_status dg_lut_conv2d4_prepared(const uint8_t *d_x4, const int8_t *d_w8, int64_t ld8, const int32_t levels[16],
                                  const dg_conv_params *p, const dg_requant *rq, void *d_out, void *d_ws, size_t ws_bytes,
                                  void *stream) {
    if (!d_x4 || !d_w8 || !levels || !p || !d_out) return DG_ERR_INVALID_ARG;
    if (p->pad_code != 0) return DG_ERR_RANGE;
    if (p->C <= 0 || p->C % 2) return DG_ERR_SHAPE;
    const int32_t wmax = max_abs16(levels);
    if (4 * wmax > 127) return DG_ERR_RANGE;
    // the same conv over 2C two-bit digit channels with identity activation levels
    dg_conv_params p2 = *p;
    p2.C = 2 * p->C;
    dg_lut lut{};
    const int32_t wl[4] = {(5 * wmax + 1) / 2, 0, 0, 0}, al[4] = {0, 1, 2, 3};   // (bound: 2 x 3 x 2.5 wmax >= 15 wmax)
    dg_status s = dg_build_lut(wl, al, 32, &lut);
    if (s != DG_OK) return s;
    return dg_lut_conv2d_prepared(d_x4, d_w8, ld8, &lut, &p2, rq, d_out, d_ws, ws_bytes, stream);
}

int64_t dg_expand_f4_ld(int64_t K) { return K <= 0 ? 0 : expand_f4_ld(K); }

dg_status dg_expand_operand_f4(const uint8_t *d_packed, int64_t rows, int64_t K, int64_t ld, const int32_t levels[4],
                               uint8_t *d_out, int64_t ld_out, void *stream) {
    if (!d_packed || !d_out || !levels) return DG_ERR_INVALID_ARG;
    if (rows < 0 || K <= 0 || ld * 4 < K || ld % 16 || ld_out < expand_f4_ld(K) || ld_out % 128) return DG_ERR_SHAPE;
    if (!aligned16(d_packed) || !aligned16(d_out)) return DG_ERR_INVALID_ARG;
    if (!tc_available()) return DG_ERR_UNSUPPORTED;
    return expand_operand_f4(d_packed, rows, K, ld, levels, d_out, ld_out, (cudaStream_t)stream);
}

dg_status dg_lut_gemm_f4(const uint8_t *d_w4, int64_t ld4, const uint8_t *d_at, int64_t lda, int64_t M, int64_t N,
                         int64_t K, const dg_lut *lut, int32_t *d_c, int64_t ldc, void *stream) {
    if (!d_w4 || !d_at || !lut || !d_c) return DG_ERR_INVALID_ARG;
    if (M <= 0 || N <= 0 || K <= 0) return DG_ERR_SHAPE;
    if (lda % 16 || lda * 4 < K || ld4 < expand_f4_ld(K) || ld4 % 128 || ldc < N) return DG_ERR_SHAPE;
    if (!aligned16(d_w4) || !aligned16(d_at)) return DG_ERR_INVALID_ARG;
    if (!lut->is_product || !tc_available()) return DG_ERR_UNSUPPORTED;
    for (int c = 0; c < 4; ++c)
        if (lut->al[c] != c || f4_nibble_half(lut->wl[c]) < 0) return DG_ERR_UNSUPPORTED;
    if ((int64_t)K * max_abs_entry(lut->entries) >= ((int64_t)1 << 22)) return DG_ERR_OVERFLOW;
    return lut_gemm_f4(d_at, lda, d_w4, ld4, M, N, K, d_c, ldc, (cudaStream_t)stream);
}

dg_status dg_lut_gemm_prepared(const uint8_t *d_w, int64_t ldw, const int8_t *d_at8, int64_t ld8,
                               int64_t M, int64_t N, int64_t K, const dg_lut *lut, void *d_c, int64_t ldc,
                               const dg_requant *rq, void *stream) {
    if (!d_w || !d_at8 || !lut || !d_c) return DG_ERR_INVALID_ARG;
    if (M <= 0 || N <= 0 || K <= 0) return DG_ERR_SHAPE;
    if (ldw % 16 || ldw * 4 < K || ld8 < expand_ld(K) || ld8 % 128) return DG_ERR_SHAPE;
    if (!aligned16(d_w) || ((uintptr_t)d_at8 & 127)) return DG_ERR_INVALID_ARG;
    if (rq ? (ldc * 4 < N) : (ldc < N)) return DG_ERR_SHAPE;
    dg_status s = check_rq(rq);
    if (s != DG_OK) return s;
    if (!lut->is_product || !levels_fit_i8(lut->wl) || !levels_fit_i8(lut->al) || !tc_available())
        return DG_ERR_UNSUPPORTED;
    if ((int64_t)K * max_abs_entry(lut->entries) >= ((int64_t)1 << 31)) return DG_ERR_OVERFLOW;
    RequantArgs a{};
    if (rq) a = to_args(rq);
    return lut_gemm_ts(d_w, ldw, d_at8, ld8, M, N, K, lut->wl, lut->al, d_c, ldc, rq ? &a : nullptr,
                       (cudaStream_t)stream, nullptr, nullptr, 0, nullptr, 0, true);
}

dg_status dg_lut_gemm_prepared_allgather(const uint8_t *d_w, int64_t ldw, const int8_t *d_at8, int64_t ld8,
                                         int64_t M, int64_t N, int64_t K, const dg_lut *lut, int32_t *d_c,
                                         int64_t ldc, int32_t *const *d_c_peers, int32_t npeers, void *stream) {
    if (!d_w || !d_at8 || !lut || !d_c || (npeers > 0 && !d_c_peers) || npeers < 0) return DG_ERR_INVALID_ARG;
    if (npeers > 7) return DG_ERR_UNSUPPORTED;
    if (M <= 0 || N <= 0 || K <= 0) return DG_ERR_SHAPE;
    if (ldw % 16 || ldw * 4 < K || ld8 < expand_ld(K) || ld8 % 128 || ldc < N) return DG_ERR_SHAPE;
    if (!aligned16(d_w) || ((uintptr_t)d_at8 & 127)) return DG_ERR_INVALID_ARG;
    for (int i = 0; i < npeers; ++i)
        if (!d_c_peers[i]) return DG_ERR_INVALID_ARG;
    if (!lut->is_product || !levels_fit_i8(lut->wl) || !levels_fit_i8(lut->al) || !tc_available())
        return DG_ERR_UNSUPPORTED;
    if ((int64_t)K * max_abs_entry(lut->entries) >= ((int64_t)1 << 31)) return DG_ERR_OVERFLOW;
    return lut_gemm_ts(d_w, ldw, d_at8, ld8, M, N, K, lut->wl, lut->al, d_c, ldc, nullptr, (cudaStream_t)stream,
                       nullptr, nullptr, 0, d_c_peers, npeers, true);
}

static bool conv_implicit_ok(const dg_conv_params *p, const uint8_t *d_x) {
    // the tensor-core kernel gathers im2col rows itself when a tap is a power-of-two number of
    // 16-byte chunks (C = 64, 128, 256, ... channels)
    const int32_t cb = p->C / 4;
    return cb >= 16 && (cb & (cb - 1)) == 0 && aligned16(d_x) && p->kh * p->kw <= 64;
}

static bool conv_is_direct(const dg_conv_params *p) {
    // a 1x1 / stride-1 / unpadded conv reads the NHWC tensor as its own im2col matrix
    return p->kh == 1 && p->kw == 1 && p->stride == 1 && p->pad == 0 && (p->C / 4) % 16 == 0;
}

// Split-K region at the tail of the conv workspace: int32 partial-sum slices [<= 8][rows][Cout],
// only for convs with few output tiles (the kernel splits K when tiles <= SMs / 2).  No
// initialisation needed: each split overwrites its slice, the reduce kernel reads them back.
static int64_t splitk_bytes(const dg_conv_params *p) {
    const int64_t Ho = (p->H + 2 * p->pad - p->kh) / p->stride + 1;
    const int64_t Wo = (p->W + 2 * p->pad - p->kw) / p->stride + 1;
    const int64_t rows = (int64_t)p->B * Ho * Wo, tiles = ((rows + 127) / 128) * ((p->Cout + 63) / 64);
    if (tiles * 2 > num_sms() * 4) return 0;   // (tile count with 64-column tiles, 4x margin)
    return (8 * rows * p->Cout * 4 + 15) / 16 * 16;   // up to 8 split slices
}

size_t dg_lut_conv2d_workspace_size(const dg_conv_params *p) {
    if (!p || p->B <= 0 || p->H <= 0 || p->W <= 0 || p->C <= 0 || p->kh <= 0 || p->kw <= 0 ||
        p->stride <= 0)
        return 0;
    const int64_t Ho = (p->H + 2 * p->pad - p->kh) / p->stride + 1;
    const int64_t Wo = (p->W + 2 * p->pad - p->kw) / p->stride + 1;
    const int64_t K = (int64_t)p->kh * p->kw * p->C;
    const int64_t rows = (int64_t)p->B * Ho * Wo;
    const int64_t cols = conv_is_direct(p) ? 0 : rows * dg_packed_ld(K);   // upper bound
    const int64_t a = (cols + 127) / 128 * 128 + (int64_t)p->Cout * expand_ld(K) + 256;
    // non-product int8 tables: one-hot activations + weight table columns after the im2col matrix
    const int64_t b = (cols + 127) / 128 * 128 + rows * onehot_ld(K) + 128 + (int64_t)p->Cout * tcols_ld(K) + 384;
    return (size_t)((a > b ? a : b) + splitk_bytes(p));
}

dg_status dg_lut_conv2d(const uint8_t *d_x, const uint8_t *d_w, const dg_lut *lut,
                        const dg_conv_params *p, const dg_requant *rq, void *d_out, void *d_ws,
                        size_t ws_bytes, int32_t variant, void *stream) {
    if (!d_x || !d_w || !lut || !p || !d_out) return DG_ERR_INVALID_ARG;
    if (variant < 0 || variant > 3) return DG_ERR_INVALID_ARG;
    if (p->B <= 0 || p->H <= 0 || p->W <= 0 || p->C <= 0 || p->Cout <= 0 || p->kh <= 0 ||
        p->kw <= 0 || p->stride <= 0 || p->pad < 0)
        return DG_ERR_SHAPE;
    if (p->C % 4 || p->pad_code < 0 || p->pad_code > 3) return DG_ERR_RANGE;
    if (rq && p->Cout % 4) return DG_ERR_SHAPE;
    const int64_t Ho = (p->H + 2 * p->pad - p->kh) / p->stride + 1;
    const int64_t Wo = (p->W + 2 * p->pad - p->kw) / p->stride + 1;
    if (Ho <= 0 || Wo <= 0) return DG_ERR_SHAPE;
    const int64_t K = (int64_t)p->kh * p->kw * p->C;
    if (p->ldw % 16 || p->ldw * 4 < K || !aligned16(d_w)) return DG_ERR_SHAPE;
    dg_status s = check_rq(rq);
    if (s != DG_OK) return s;
    if (K * max_abs_entry(lut->entries) >= ((int64_t)1 << 31)) return DG_ERR_OVERFLOW;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t rows = (int64_t)p->B * Ho * Wo;
    const bool tc_ok = lut->is_product && levels_fit_i8(lut->wl) && levels_fit_i8(lut->al) && tc_available();
    if ((variant == 0 || variant == 2) && tc_ok && !conv_is_direct(p) && conv_implicit_ok(p, d_x)) {
        // implicit GEMM: no im2col matrix; weights expanded into the workspace
        const int64_t ld8 = expand_ld(K);
        int8_t *w8 = (int8_t *)(((uintptr_t)d_ws + 127) & ~(uintptr_t)127);
        if (!d_ws || (int64_t)ws_bytes - (int64_t)((uint8_t *)w8 - (uint8_t *)d_ws) < p->Cout * ld8) return DG_ERR_WORKSPACE;
        s = expand_operand(d_w, p->Cout, K, p->ldw, lut->wl, w8, ld8, st);
        if (s != DG_OK) return s;
        RequantArgs ra{};
        if (rq) ra = to_args(rq);
        TsConv cv{d_x, p->H, p->W, p->C / 4, p->kh, p->kw, p->stride, p->pad, (int32_t)Ho, (int32_t)Wo, p->pad_code};
        return lut_gemm_ts(nullptr, 0, w8, ld8, rows, p->Cout, K, lut->al, lut->wl, d_out, rq ? p->Cout / 4 : p->Cout,
                           rq ? &ra : nullptr, st, &cv);
    }
    const uint8_t *P;
    int64_t ldp;
    if (conv_is_direct(p) && aligned16(d_x)) {
        P = d_x;
        ldp = p->C / 4;
    } else {
        const int64_t ld = dg_packed_ld(K);
        if (!d_ws || (int64_t)ws_bytes < rows * ld) return DG_ERR_WORKSPACE;
        uint8_t *cols = (uint8_t *)(((uintptr_t)d_ws + 127) & ~(uintptr_t)127);
        if ((int64_t)ws_bytes - (int64_t)(cols - (uint8_t *)d_ws) < rows * ld) return DG_ERR_WORKSPACE;
        s = dg_im2col(d_x, p->B, p->H, p->W, p->C, p->kh, p->kw, p->stride, p->pad,
                      (uint8_t)p->pad_code, cols, ld, stream);
        if (s != DG_OK) return s;
        P = cols;
        ldp = ld;
    }
    // P = pixels (activation codes), Q = weights: D[pixel][cout] is the NHWC output; the
    // table is transposed so that the index stays (w<<2)|a: Tt[(a<<2)|w] = T[(w<<2)|a].
    int32_t Tt[16];
    for (int a = 0; a < 4; ++a)
        for (int w = 0; w < 4; ++w) Tt[(a << 2) | w] = lut->entries[(w << 2) | a];
    const int64_t ldd = rq ? p->Cout / 4 : p->Cout;
    // the rest of the workspace (after the im2col matrix) holds the expanded operands
    uint8_t *ws_rest = (uint8_t *)d_ws;
    size_t rest = ws_bytes;
    if (P != d_x) {
        const int64_t used = (int64_t)(((uintptr_t)P - (uintptr_t)d_ws) + rows * ldp);
        ws_rest = (uint8_t *)d_ws + used;
        rest = ws_bytes > (size_t)used ? ws_bytes - (size_t)used : 0;
    }
    return gemm_dispatch(P, ldp, d_w, p->ldw, rows, p->Cout, K, Tt, lut->is_product != 0, lut->al,
                         lut->wl, d_out, ldd, rq, ws_rest, rest, variant, st);
}

dg_status dg_lut_conv2d_prepared(const uint8_t *d_x, const int8_t *d_w8, int64_t ld8, const dg_lut *lut,
                                 const dg_conv_params *p, const dg_requant *rq, void *d_out, void *d_ws, size_t ws_bytes,
                                 void *stream) {
    if (!d_x || !d_w8 || !lut || !p || !d_out) return DG_ERR_INVALID_ARG;
    if (p->B <= 0 || p->H <= 0 || p->W <= 0 || p->C <= 0 || p->Cout <= 0 || p->kh <= 0 || p->kw <= 0 ||
        p->stride <= 0 || p->pad < 0)
        return DG_ERR_SHAPE;
    if (p->C % 4 || p->pad_code < 0 || p->pad_code > 3) return DG_ERR_RANGE;
    if (rq && p->Cout % 4) return DG_ERR_SHAPE;
    const int64_t Ho = (p->H + 2 * p->pad - p->kh) / p->stride + 1;
    const int64_t Wo = (p->W + 2 * p->pad - p->kw) / p->stride + 1;
    if (Ho <= 0 || Wo <= 0) return DG_ERR_SHAPE;
    const int64_t K = (int64_t)p->kh * p->kw * p->C;
    if (ld8 < expand_ld(K) || ld8 % 128 || ((uintptr_t)d_w8 & 127)) return DG_ERR_SHAPE;
    dg_status s = check_rq(rq);
    if (s != DG_OK) return s;
    if (!lut->is_product || !levels_fit_i8(lut->wl) || !levels_fit_i8(lut->al) || !tc_available())
        return DG_ERR_UNSUPPORTED;
    if (K * max_abs_entry(lut->entries) >= ((int64_t)1 << 31)) return DG_ERR_OVERFLOW;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t rows = (int64_t)p->B * Ho * Wo;
    RequantArgs ra{};
    if (rq) ra = to_args(rq);
    const int64_t ldd = rq ? p->Cout / 4 : p->Cout;
    // (direct / implicit paths: d_ws, if given, serves split-K; it must be zero and is left zero)
    const int64_t skb = splitk_bytes(p);
    void *skws = nullptr;
    if (d_ws && skb > 0 && (int64_t)ws_bytes >= skb) {
        const uintptr_t tail = ((uintptr_t)d_ws + ws_bytes - (size_t)skb) & ~(uintptr_t)15;
        if (tail >= (uintptr_t)d_ws) skws = reinterpret_cast<void *>(tail);
    }
    if (conv_is_direct(p) && aligned16(d_x))
        return lut_gemm_ts(d_x, p->C / 4, d_w8, ld8, rows, p->Cout, K, lut->al, lut->wl, d_out, ldd, rq ? &ra : nullptr, st,
                           nullptr, skws, (size_t)skb, nullptr, 0, true);
    if (conv_implicit_ok(p, d_x)) {
        TsConv cv{d_x, p->H, p->W, p->C / 4, p->kh, p->kw, p->stride, p->pad, (int32_t)Ho, (int32_t)Wo, p->pad_code};
        return lut_gemm_ts(nullptr, 0, d_w8, ld8, rows, p->Cout, K, lut->al, lut->wl, d_out, ldd, rq ? &ra : nullptr, st,
                           &cv, skws, (size_t)skb, nullptr, 0, true);
    }
    // explicit im2col fallback (e.g. VGG conv1_1 with C = 4 padded channels)
    const int64_t ld = dg_packed_ld(K);
    uint8_t *cols = (uint8_t *)(((uintptr_t)d_ws + 127) & ~(uintptr_t)127);
    if (!d_ws || (int64_t)ws_bytes - (int64_t)(cols - (uint8_t *)d_ws) < rows * ld) return DG_ERR_WORKSPACE;
    s = dg_im2col(d_x, p->B, p->H, p->W, p->C, p->kh, p->kw, p->stride, p->pad, (uint8_t)p->pad_code, cols, ld, stream);
    if (s != DG_OK) return s;
    return lut_gemm_ts(cols, ld, d_w8, ld8, rows, p->Cout, K, lut->al, lut->wl, d_out, ldd, rq ? &ra : nullptr, st,
                       nullptr, nullptr, 0, nullptr, 0, true);
}

}  // extern "C"
