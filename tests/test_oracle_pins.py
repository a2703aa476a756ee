"""Pins of the CPU oracle against things other than itself (no GPU needed).

Each test names the passage / mathematical fact it pins.  A plausible mistake
in oracle.c (dropped term, swapped w/a in the index, wrong shift, wrong tie
rule, wrong padding) fails at least one of them:
  * index order w<<2|a        -> non-symmetric tables in test_gemm_closed_form / brute force
  * dropped k / off-by-one K  -> one-hot-table count test, K-split additivity
  * transposed operand        -> non-square closed-form shapes
  * padding                   -> border-count test and pad_code im2col test
  * requant tie / sign rule   -> exact Fraction sweep over all ties
"""
import itertools
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                yield line


def _ints(s, sep=","):
    return [int(v) for v in s.split(sep) if v.strip()]


def _pack_np(codes):
    """Independent packer for tests: byte j = sum_i codes[4j+i] << 2i."""
    codes = np.asarray(codes, np.uint8)
    rows, K = codes.shape
    Kp = (K + 3) // 4 * 4
    c = np.zeros((rows, Kp), np.uint16)
    c[:, :K] = codes
    c = c.reshape(rows, Kp // 4, 4)
    return (c[..., 0] | (c[..., 1] << 2) | (c[..., 2] << 4) | (c[..., 3] << 6)).astype(np.uint8)


# ---------------------------------------------------------------- packing
def test_unpack_golden():
    for line in _rows("pack_examples.txt"):
        codes_s, bytes_s = line.split("->")
        codes = _ints(codes_s)
        packed = np.array([int(b, 16) for b in bytes_s.split()], np.uint8)
        got = oracle.unpack_codes(packed, 1, len(codes), len(packed))
        assert got.tolist() == [codes], line


@pytest.mark.parametrize("K", [1, 3, 4, 5, 17, 64, 131])
def test_unpack_roundtrip_random(K):
    g = np.random.default_rng(K)
    codes = g.integers(0, 4, size=(7, K), dtype=np.uint8)
    packed = _pack_np(codes)
    ld = packed.shape[1] + 16          # leading dimension larger than the row
    buf = np.zeros((7, ld), np.uint8)
    buf[:, :packed.shape[1]] = packed
    assert np.array_equal(oracle.unpack_codes(buf, 7, K, ld), codes)


# ---------------------------------------------------------------- LUT-16
def test_lut16_golden():
    for line in _rows("lut16_examples.txt"):
        wl_s, al_s, pairs, mm = [p.strip() for p in line.split(";")]
        T = oracle.build_lut16(_ints(wl_s), _ints(al_s))
        for kv in pairs.split():
            k, v = kv.split("=")
            assert T[int(k)] == int(v), (line, kv)
        mx, mn = [int(x.split("=")[1]) for x in mm.split()]
        assert T.max() == mx and T.min() == mn


def test_lut16_is_outer_product_and_table2_size():
    g = np.random.default_rng(1)
    for _ in range(50):
        wl = g.integers(-127, 128, 4)
        al = g.integers(-127, 128, 4)
        T = oracle.build_lut16(wl, al)
        # row index = weight code (high 2 bits), column = activation code (Q7)
        assert np.array_equal(T.reshape(4, 4), np.outer(wl, al))
    # Table 2: 2-bit -> 4-bit index -> 16 entries -> 128 bits at int8
    T = oracle.build_lut16([-2, -1, 0, 1], [0, 1, 2, 3])
    assert T.size == 16 and T.astype(np.int8).nbytes * 8 == 128
    assert np.array_equal(T.astype(np.int8).astype(np.int32), T)


# ---------------------------------------------------------------- GEMM
def test_gemm_golden():
    for line in _rows("gemm_examples.txt"):
        wl_s, al_s, w_s, a_s, c_s = [p.strip() for p in line.split(";")]
        T = oracle.build_lut16(_ints(wl_s), _ints(al_s))
        W = np.array([_ints(w_s)], np.uint8)
        A = np.array(_ints(a_s), np.uint8).reshape(-1, 1)
        assert oracle.lut_gemm(W, A, T)[0, 0] == int(c_s)


def test_gemm_closed_form_fp64_blas():
    """For a product table, C = WL @ AL with dequantised integer levels; fp64 BLAS is
    exact here (all partial sums are integers << 2^53).  S:529: >=500 random
    instances with M,N,K in [1,64]."""
    g = np.random.default_rng(2)
    for it in range(500):
        M, N, K = g.integers(1, 65, 3)
        wl = g.integers(-8, 8, 4)
        al = g.integers(-8, 8, 4)
        W = g.integers(0, 4, (M, K), dtype=np.uint8)
        A = g.integers(0, 4, (K, N), dtype=np.uint8)
        T = oracle.build_lut16(wl, al)
        C = oracle.lut_gemm(W, A, T)
        ref = wl[W].astype(np.float64) @ al[A].astype(np.float64)
        assert np.array_equal(C, ref.astype(np.int64)), it


def test_gemm_closed_form_config1_shape():
    """BJ configs[0]: M=64, N=196, K=576, wl={-2..1}, al={0..3}."""
    g = np.random.default_rng(3)
    W = g.integers(0, 4, (64, 576), dtype=np.uint8)
    A = g.integers(0, 4, (576, 196), dtype=np.uint8)
    wl, al = np.array([-2, -1, 0, 1]), np.array([0, 1, 2, 3])
    C = oracle.lut_gemm(W, A, oracle.build_lut16(wl, al))
    assert np.array_equal(C, (wl[W].astype(np.float64) @ al[A].astype(np.float64)).astype(np.int64))


@pytest.mark.parametrize("K", [1, 2, 3, 4])
def test_gemm_brute_force_all_assignments(K):
    """Every weight code vector against every activation code vector (4^K x 4^K), for a
    random NON-product table, against the one-hot count decomposition
    C[m][n] = sum_{i,j} T[i][j] * #{k : W[m][k]=i and A[k][n]=j}."""
    g = np.random.default_rng(10 + K)
    T = g.integers(-1000, 1000, 16).astype(np.int32)
    vecs = np.array(list(itertools.product(range(4), repeat=K)), np.uint8)  # [4^K][K]
    W = vecs
    A = np.ascontiguousarray(vecs.T)
    C = oracle.lut_gemm(W, A, T)
    ohW = np.eye(4, dtype=np.int64)[W]          # [m][k][i]
    ohA = np.eye(4, dtype=np.int64)[A]          # [k][n][j]
    counts = np.einsum("mki,knj->mnij", ohW, ohA)
    assert np.array_equal(C, np.einsum("mnij,ij->mn", counts, T.reshape(4, 4).astype(np.int64)))


def test_gemm_invariants():
    g = np.random.default_rng(4)
    M, N, K = 9, 13, 37
    W = g.integers(0, 4, (M, K), dtype=np.uint8)
    A = g.integers(0, 4, (K, N), dtype=np.uint8)
    T1 = g.integers(-500, 500, 16).astype(np.int32)
    T2 = g.integers(-500, 500, 16).astype(np.int32)
    G = lambda T, W=W, A=A: oracle.lut_gemm(W, A, T).astype(np.int64)
    # linearity in the table
    assert np.array_equal(G(T1 + T2), G(T1) + G(T2))
    assert np.array_equal(G(3 * T1), 3 * G(T1))
    # one-hot tables count every (m,n,k) pair exactly once
    tot = sum(G(np.eye(16, dtype=np.int32)[e]) for e in range(16))
    assert np.all(tot == K)
    # all-zero activation levels (code 0 with al[0]=0) -> 0 (BJ north_star)
    Tp = oracle.build_lut16([-2, -1, 0, 1], [0, 1, 2, 3])
    assert np.all(G(Tp, A=np.zeros_like(A)) == 0)
    # zero-level weights (code 2 with wl[2]=0) -> 0
    assert np.all(G(Tp, W=np.full_like(W, 2)) == 0)
    # K-split additivity
    k1 = 11
    assert np.array_equal(G(T1), G(T1, W=W[:, :k1], A=A[:k1]) + G(T1, W=W[:, k1:], A=A[k1:]))
    # common permutation of K leaves C unchanged
    p = g.permutation(K)
    assert np.array_equal(G(T1), G(T1, W=W[:, p], A=A[p]))
    # M / N concatenation
    assert np.array_equal(G(T1)[:4], G(T1, W=W[:4]))
    assert np.array_equal(G(T1)[:, 5:], G(T1, A=A[:, 5:]))


def test_gemm_overflow_detected():
    T = np.full(16, 1 << 30, np.int32)
    W = np.zeros((1, 4), np.uint8)
    A = np.zeros((4, 1), np.uint8)
    with pytest.raises(OverflowError):
        oracle.lut_gemm(W, A, T)


# ---------------------------------------------------------------- conv
def _im2col_np(x, kh, kw, stride, pad, pad_code):
    """Test-side im2col (numpy), independent of oracle.conv2d_direct."""
    B, H, Wd, C = x.shape
    xp = np.full((B, H + 2 * pad, Wd + 2 * pad, C), pad_code, np.uint8)
    xp[:, pad:pad + H, pad:pad + Wd] = x
    Ho = (H + 2 * pad - kh) // stride + 1
    Wo = (Wd + 2 * pad - kw) // stride + 1
    cols = np.empty((B, Ho, Wo, kh, kw, C), np.uint8)
    for r in range(kh):
        for s in range(kw):
            cols[:, :, :, r, s] = xp[:, r:r + stride * Ho:stride, s:s + stride * Wo:stride]
    return cols.reshape(B * Ho * Wo, kh * kw * C), (B, Ho, Wo)


def test_conv_1x1_is_gemm():
    g = np.random.default_rng(5)
    x = g.integers(0, 4, (2, 5, 6, 12), dtype=np.uint8)
    w = g.integers(0, 4, (7, 1, 1, 12), dtype=np.uint8)
    T = g.integers(-50, 50, 16).astype(np.int32)
    out = oracle.conv2d_direct(x, w, T, stride=1, pad=0)
    C = oracle.lut_gemm(w.reshape(7, 12), np.ascontiguousarray(x.reshape(-1, 12).T), T)
    assert np.array_equal(out.reshape(-1, 7), C.T)


def test_conv_border_counts():
    """3x3, pad 1, every in-image product = 1 and pad level 0: interior 9*Cin,
    edges 6*Cin, corners 4*Cin (pins the padding)."""
    Cin = 5
    x = np.ones((1, 6, 7, Cin), np.uint8)                # code 1 -> level 1
    w = np.zeros((2, 3, 3, Cin), np.uint8)               # code 0 -> level 1
    T = oracle.build_lut16([1, 1, 1, 1], [0, 1, 1, 1])   # pad code 0 -> level 0
    out = oracle.conv2d_direct(x, w, T, stride=1, pad=1, pad_code=0)[0, :, :, 0]
    exp = np.full((6, 7), 9 * Cin)
    exp[0, :] = exp[-1, :] = exp[:, 0] = exp[:, -1] = 6 * Cin
    exp[0, 0] = exp[0, -1] = exp[-1, 0] = exp[-1, -1] = 4 * Cin
    assert np.array_equal(out, exp)


@pytest.mark.parametrize("k,stride,pad,pad_code", [(3, 1, 1, 0), (3, 2, 1, 0), (1, 2, 0, 0),
                                                   (3, 1, 1, 2), (5, 2, 2, 3)])
def test_conv_vs_im2col_histogram(k, stride, pad, pad_code):
    """Direct conv vs (numpy im2col + one-hot count decomposition) for a non-product table."""
    g = np.random.default_rng(100 + k * 10 + stride + pad_code)
    x = g.integers(0, 4, (2, 9, 8, 6), dtype=np.uint8)
    w = g.integers(0, 4, (5, k, k, 6), dtype=np.uint8)
    T = g.integers(-99, 99, 16).astype(np.int32)
    out = oracle.conv2d_direct(x, w, T, stride=stride, pad=pad, pad_code=pad_code)
    cols, (B, Ho, Wo) = _im2col_np(x, k, k, stride, pad, pad_code)
    Wm = w.reshape(5, -1)
    ohW = np.eye(4, dtype=np.int64)[Wm]
    ohA = np.eye(4, dtype=np.int64)[cols]
    counts = np.einsum("mki,nkj->nmij", ohW, ohA)
    ref = np.einsum("nmij,ij->nm", counts, T.reshape(4, 4).astype(np.int64))
    assert np.array_equal(out.reshape(-1, 5), ref)


def test_conv_closed_form_fp64():
    g = np.random.default_rng(6)
    wl, al = np.array([-2, -1, 0, 1]), np.array([0, 1, 2, 3])
    x = g.integers(0, 4, (3, 7, 7, 8), dtype=np.uint8)
    w = g.integers(0, 4, (16, 3, 3, 8), dtype=np.uint8)
    out = oracle.conv2d_direct(x, w, oracle.build_lut16(wl, al), stride=2, pad=1, pad_code=0)
    cols, _ = _im2col_np(x, 3, 3, 2, 1, 0)
    ref = al[cols].astype(np.float64) @ wl[w.reshape(16, -1)].astype(np.float64).T
    assert np.array_equal(out.reshape(-1, 16), ref.astype(np.int64))


# ---------------------------------------------------------------- requant
def _req_exact(v, mult, shift, zp, qmin, qmax):
    x = Fraction(v * mult, 1 << shift)
    # round half away from zero on exact rationals
    r = int(abs(x) + Fraction(1, 2)) * (1 if x >= 0 else -1)
    return min(max(r + zp, qmin), qmax)


@pytest.mark.parametrize("shift", [1, 7, 20, 31])
def test_requant_exact_fraction(shift):
    g = np.random.default_rng(shift)
    accs = np.arange(-3000, 3001, dtype=np.int32)
    params = [(1 << (shift - 1), 0, 0, -2, 1),            # mult = 2^(s-1): every odd v is a tie
              (int(g.integers(1, 1 << 16)), 0, 1, 0, 3),
              (int(g.integers(1, 1 << 20)), -1, 2, -8, 7),
              (-int(g.integers(1, 1 << 12)), 0, 0, 0, 3)]
    for mult, bias, zp, qmin, qmax in params:
        bias_v = np.array([bias], np.int32)
        got = oracle.requantize(accs.reshape(-1, 1), mult, shift, zp, qmin, qmax, bias=bias_v)
        exp = [_req_exact(int(a) + bias, mult, shift, zp, qmin, qmax) for a in accs]
        # codes are returned as one byte each; negative codes are two's-complement bytes
        assert got[:, 0].view(np.int8).astype(np.int64).tolist() == exp, (mult, bias, zp)


def test_requant_residual_and_bias_axes():
    g = np.random.default_rng(7)
    acc = g.integers(-5000, 5000, (6, 10)).astype(np.int32)
    res = g.integers(-500, 500, (6, 10)).astype(np.int32)
    bcol = g.integers(-100, 100, 10).astype(np.int32)
    brow = g.integers(-100, 100, 6).astype(np.int32)
    mult, shift, zp = 20180, 20, 1
    got0 = oracle.requantize(acc, mult, shift, zp, 0, 3, res=res, bias=bcol, bias_axis=0)
    got1 = oracle.requantize(acc, mult, shift, zp, 0, 3, res=res, bias=brow, bias_axis=1)
    for r in range(6):
        for c in range(10):
            assert got0[r, c] == _req_exact(int(acc[r, c]) + int(res[r, c]) + int(bcol[c]), mult, shift, zp, 0, 3)
            assert got1[r, c] == _req_exact(int(acc[r, c]) + int(res[r, c]) + int(brow[r]), mult, shift, zp, 0, 3)


def test_requant_config1_not_degenerate():
    """Q12: with bias 432, mult 20180, zp 1 the config-1 code histogram is spread."""
    import synth
    g = np.random.default_rng(8)
    W = g.integers(0, 4, (64, 576), dtype=np.uint8)
    A = g.integers(0, 4, (576, 196), dtype=np.uint8)
    C = oracle.lut_gemm(W, A, oracle.build_lut16([-2, -1, 0, 1], [0, 1, 2, 3]))
    rq = synth.CFG1_RQ
    assert (rq.bias, rq.mult, rq.zp) == (432, 20180, 1)
    codes = oracle.requantize(C, rq.mult, rq.shift, rq.zp, 0, 3, bias=np.full(64, rq.bias, np.int32),
                              bias_axis=1)
    hist = np.bincount(codes.ravel(), minlength=4) / codes.size
    assert np.all(hist > 0.02), hist


# ---------------------------------------------------------------- Eq. 1
def test_quantize_golden():
    for line in _rows("quantize_examples.txt"):
        x, s, z, qmin, qmax, exp = [p.strip() for p in line.split(";")]
        q = oracle.quantize(np.array([float(x)], np.float32), float(s), float(z), int(qmin), int(qmax))
        assert q[0] == int(exp), line


def test_quantize_properties():
    g = np.random.default_rng(9)
    x = np.sort(g.uniform(-3, 3, 4000).astype(np.float32))
    s, z = 1.7, 0.25
    q = oracle.quantize(x, s, z, -2, 1)
    assert np.all(np.diff(q) >= 0)                 # monotone
    assert q.min() >= -2 and q.max() <= 1          # inside clip range
    inside = (s * x + z > -2.5) & (s * x + z < 1.5)
    err = np.abs(x[inside] - (q[inside] - z) / s)  # roundtrip bound 0.5/|s|
    assert np.all(err <= 0.5 / s + 1e-6)


# ---------------------------------------------------------------- Freivalds
def test_freivalds_accepts_truth_rejects_fault():
    g = np.random.default_rng(11)
    M, N, K = 20, 33, 41
    W = g.integers(0, 4, (M, K), dtype=np.uint8)
    At = g.integers(0, 4, (N, K), dtype=np.uint8)
    T = g.integers(-16129, 16130, 16).astype(np.int32)
    C = oracle.lut_gemm(W, np.ascontiguousarray(At.T), T)
    assert oracle.freivalds_rows(W, At, C, T) == 0
    for (m, n) in [(0, 0), (7, 32), (19, 13)]:
        Cb = C.copy()
        Cb[m, n] += 1
        assert oracle.freivalds_rows(W, At, Cb, T) > 0


# ---- b-bit LUT GEMM (Table 2) -----------------------------------------
@pytest.mark.parametrize("bits", [2, 3, 4])
def test_gemm_bits_closed_form_fp64(bits):
    """Product tables T[(i<<b)|j] = wl[i]*al[j] (2^(2b) entries, Table 2): C = WL @ AL in fp64
    (exact: integer partial sums << 2^53), random shapes and level sets."""
    g = np.random.default_rng(20 + bits)
    L = 1 << bits
    for it in range(60):
        M, N, K = g.integers(1, 40, 3)
        wl = g.integers(-40, 41, L)
        al = g.integers(-40, 41, L)
        T = np.outer(wl, al).reshape(-1).astype(np.int32)     # index (i << b) | j, row-major
        W = g.integers(0, L, (M, K), dtype=np.uint8)
        A = g.integers(0, L, (K, N), dtype=np.uint8)
        C = oracle.lut_gemm_bits(W, A, T, bits)
        assert np.array_equal(C, (wl[W].astype(np.float64) @ al[A].astype(np.float64)).astype(np.int64)), it


@pytest.mark.parametrize("bits,K", [(3, 1), (3, 2), (4, 1), (4, 2)])
def test_gemm_bits_brute_force_non_product(bits, K):
    """Every b-bit weight vector x every b-bit activation vector (2^(bK) x 2^(bK)) for a random
    NON-product 2^(2b)-entry table, against the pair-count decomposition
    C[m][n] = sum_{i,j} T[i][j] #{k : W[m][k] = i, A[k][n] = j}."""
    g = np.random.default_rng(30 + 10 * bits + K)
    L = 1 << bits
    T = g.integers(-1000, 1000, L * L).astype(np.int32)
    vecs = np.array(list(itertools.product(range(L), repeat=K)), np.uint8)
    C = oracle.lut_gemm_bits(vecs, np.ascontiguousarray(vecs.T), T, bits)
    ohW = np.eye(L, dtype=np.int64)[vecs]
    ohA = np.eye(L, dtype=np.int64)[np.ascontiguousarray(vecs.T)]
    counts = np.einsum("mki,knj->mnij", ohW, ohA)
    assert np.array_equal(C, np.einsum("mnij,ij->mn", counts, T.reshape(L, L).astype(np.int64)))


def test_gemm_bits_index_order_and_digit_split():
    """The weight code is the HIGH part of the index (a transposed table changes the result), and a
    4-bit activation code a = 4 a_h + a_l with identity levels splits into two 2-bit digit GEMMs:
    C = G2(W, A_l; wl x {0,1,2,3}) + 4 G2(W, A_h; wl x {0,1,2,3}) for 2-bit W."""
    g = np.random.default_rng(41)
    M, N, K = 7, 9, 33
    T = g.integers(-50, 50, 256).astype(np.int32)
    W = g.integers(0, 16, (M, K), dtype=np.uint8)
    A = g.integers(0, 16, (K, N), dtype=np.uint8)
    Tt = T.reshape(16, 16).T.reshape(-1).copy()
    assert not np.array_equal(oracle.lut_gemm_bits(W, A, T, 4), oracle.lut_gemm_bits(W, A, Tt, 4))
    # digit split against the independently pinned 2-bit oracle
    wl = g.integers(-20, 20, 16)
    W2 = g.integers(0, 4, (M, K), dtype=np.uint8)
    wl2 = wl[:4]
    T4 = np.outer(np.concatenate([wl2, np.zeros(12, np.int64)]), np.arange(16)).reshape(-1).astype(np.int32)
    Tid = oracle.build_lut16(wl2, [0, 1, 2, 3])
    lhs = oracle.lut_gemm_bits(W2, A, T4, 4)
    rhs = oracle.lut_gemm(W2, A & 3, Tid).astype(np.int64) + 4 * oracle.lut_gemm(W2, A >> 2, Tid).astype(np.int64)
    assert np.array_equal(lhs, rhs)


@pytest.mark.parametrize("bits", [2, 4])
def test_conv_bits_against_pinned_routes(bits):
    """The b-bit direct conv: at b = 2 it equals the pinned 2-bit direct conv (same T); at b = 4 a
    1x1 stride-1 conv equals the pinned b-bit GEMM, and a 3x3 conv with every level 1 counts the
    in-image taps (9 / 6 / 4 x C at interior / edge / corner pixels, pad code 0 = level 0)."""
    g = np.random.default_rng(50 + bits)
    L = 1 << bits
    T = g.integers(-300, 300, L * L).astype(np.int32)
    x = g.integers(0, L, (2, 6, 5, 3), dtype=np.uint8)
    w = g.integers(0, L, (4, 3, 3, 3), dtype=np.uint8)
    got = oracle.conv2d_direct_bits(x, w, T, 1, 1, bits, pad_code=1)
    if bits == 2:
        assert np.array_equal(got, oracle.conv2d_direct(x, w, T, 1, 1, pad_code=1))
        return
    w1 = g.integers(0, L, (5, 1, 1, 3), dtype=np.uint8)
    c1 = oracle.conv2d_direct_bits(x, w1, T, 1, 0, bits).reshape(-1, 5)
    assert np.array_equal(c1, oracle.lut_gemm_bits(w1.reshape(5, 3), np.ascontiguousarray(x.reshape(-1, 3).T), T, bits).T)
    ones = np.zeros(256, np.int32)
    ones[(np.arange(16)[:, None] << 4 | np.arange(1, 16)[None, :]).reshape(-1)] = 1   # level 1 unless a = 0
    xs = g.integers(1, 16, (1, 5, 5, 2), dtype=np.uint8)
    ws = g.integers(0, 16, (1, 3, 3, 2), dtype=np.uint8)
    cnt = oracle.conv2d_direct_bits(xs, ws, ones, 1, 1, bits)[0, :, :, 0]
    assert cnt[2, 2] == 18 and cnt[0, 2] == 12 and cnt[0, 0] == 8


# ---------------------------------------------------------------- whole-output conv Freivalds
CONV_FV = [  # B, H, W, C, Cout, k, stride, pad, pad_code
    (2, 7, 6, 5, 4, 3, 1, 1, 0), (1, 9, 9, 8, 3, 3, 2, 1, 2), (2, 5, 7, 4, 6, 1, 2, 0, 0),
    (1, 8, 8, 3, 5, 5, 1, 2, 3), (3, 6, 6, 4, 2, 3, 1, 1, 1), (1, 11, 10, 4, 3, 7, 2, 3, 0),
]


@pytest.mark.parametrize("B,H,W,C,Cout,k,stride,pad,pad_code", CONV_FV)
def test_conv_freivalds_accepts_truth_rejects_every_single_fault(B, H, W, C, Cout, k, stride, pad, pad_code):
    """or_conv_freivalds against the pinned direct conv: the true output
    passes for any table, stride, padding and pad code; a +-1 fault at EVERY output element, a
    swap of two channels and a swap of two pixels are each caught (r[p] is never 0)."""
    g = np.random.default_rng(B * 100 + H * 10 + k + pad_code)
    x = g.integers(0, 4, (B, H, W, C), dtype=np.uint8)
    w = g.integers(0, 4, (Cout, k, k, C), dtype=np.uint8)
    T = g.integers(-50, 51, 16).astype(np.int32)          # non-product table
    out = oracle.conv2d_direct(x, w, T, stride, pad, pad_code).reshape(-1, Cout)
    assert oracle.conv_freivalds(x, w, T, stride, pad, pad_code, out, trials=2) == 0
    for p in range(out.shape[0]):
        for co in range(Cout):
            bad = out.copy()
            bad[p, co] += 1 if (p + co) % 2 else -1
            assert oracle.conv_freivalds(x, w, T, stride, pad, pad_code, bad, seed=p) == 1, (p, co)
    sw = out.copy()
    sw[:, [0, 1]] = sw[:, [1, 0]]
    if not np.array_equal(sw, out):
        assert oracle.conv_freivalds(x, w, T, stride, pad, pad_code, sw) >= 1
    sp = out.copy()
    sp[[0, -1]] = sp[[-1, 0]]
    if not np.array_equal(sp, out):
        assert oracle.conv_freivalds(x, w, T, stride, pad, pad_code, sp) >= 1
    # the pad code matters wherever a tap leaves the image: a wrong pad code is rejected
    if pad > 0:
        assert oracle.conv_freivalds(x, w, T, stride, pad, (pad_code + 1) % 4, out) >= 1


def test_conv_freivalds_1x1_agrees_with_gemm_freivalds():
    """A 1x1 / stride-1 conv is the GEMM C^T = LUTGEMM(W, X^T): both whole-output checks
    accept the truth and reject the same injected fault."""
    g = np.random.default_rng(12)
    B, H, W, C, Cout = 2, 5, 6, 9, 7
    x = g.integers(0, 4, (B, H, W, C), dtype=np.uint8)
    w = g.integers(0, 4, (Cout, 1, 1, C), dtype=np.uint8)
    T = oracle.build_lut16([-2, -1, 0, 1], [0, 1, 2, 3])
    out = oracle.conv2d_direct(x, w, T, 1, 0, 0).reshape(-1, Cout)
    Wm, Xt = w.reshape(Cout, C), x.reshape(-1, C)
    assert oracle.conv_freivalds(x, w, T, 1, 0, 0, out) == 0
    assert oracle.freivalds_rows(Wm, Xt, np.ascontiguousarray(out.T), T) == 0
    out[3, 4] += 7
    assert oracle.conv_freivalds(x, w, T, 1, 0, 0, out) == 1
    assert oracle.freivalds_rows(Wm, Xt, np.ascontiguousarray(out.T), T) >= 1


# ---------------------------------------------------------------- float-valued tables
def test_gemm_f64_float_product_table_closed_form():
    """A float PRODUCT table T = wl (x) al (non-uniform quantiser levels) makes the LUT
    sum the dense product of the level matrices: equal to fp64 BLAS within its rounding."""
    g = np.random.default_rng(31)
    for M, N, K in [(7, 5, 33), (16, 40, 300), (3, 64, 1000)]:
        wl, al = g.normal(size=4), np.abs(g.normal(size=4))
        T = np.outer(wl, al).reshape(-1)          # index (i << 2) | j
        W = g.integers(0, 4, (M, K), dtype=np.uint8)
        A = g.integers(0, 4, (K, N), dtype=np.uint8)
        C = oracle.lut_gemm_f64(W, A, T)
        ref = wl[W] @ al[A]
        assert np.allclose(C, ref, rtol=0, atol=K * 4e-15 * np.abs(T).max())
        # the transposed index (a << 2 | w) would give a different result for asymmetric levels
        Tt = np.outer(wl, al).T.reshape(-1)
        assert not np.allclose(oracle.lut_gemm_f64(W, A, Tt), ref)


def test_gemm_f64_integer_table_equals_integer_oracle_and_pair_counts():
    """Integer-valued float tables reproduce the pinned integer oracle exactly; any table equals the
    pair-count form sum_{i,j} T[(i<<2)|j] * #{k : W=i, A=j} (brute force over the counts)."""
    g = np.random.default_rng(32)
    M, N, K = 9, 11, 257
    W = g.integers(0, 4, (M, K), dtype=np.uint8)
    A = g.integers(0, 4, (K, N), dtype=np.uint8)
    Ti = g.integers(-1000, 1000, 16).astype(np.int32)
    assert np.array_equal(oracle.lut_gemm_f64(W, A, Ti.astype(np.float64)), oracle.lut_gemm(W, A, Ti).astype(np.float64))
    Tf = g.normal(size=16) * 10.0 ** g.integers(-3, 4, 16)
    cnt = np.zeros((M, N, 16))
    for i in range(4):
        for j in range(4):
            cnt[:, :, (i << 2) | j] = (W == i).astype(np.float64) @ (A == j).astype(np.float64)
    assert np.allclose(oracle.lut_gemm_f64(W, A, Tf), cnt @ Tf, rtol=1e-12, atol=1e-9)
