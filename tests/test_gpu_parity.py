"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit-exact.

Every output is integer (codes, int32 accumulators), so the bar is exact equality
(DESIGN.md §4).  Inputs come from seeded generators; expected values come only from
oracle/.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2304_09049_b200 import dg  # noqa: E402

DEV = "cuda"
VARIANTS = ["cc", "tc", "tc_ss"]
WL, AL = [-2, -1, 0, 1], [0, 1, 2, 3]


def gpu_pack(codes_np, weights=False):
    c = torch.from_numpy(np.ascontiguousarray(codes_np, dtype=np.uint8)).to(DEV)
    return dg.pack_codes(c, weights=weights)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def oracle_codes_of(packed_gpu, rows, K):
    p = host(packed_gpu)
    return oracle.unpack_codes(p, rows, K, p.shape[1])


def variant_ok(variant, lut):
    if variant.startswith("tc") and not (lut.is_product and dg.lib() and _tc_available()):
        return False
    return True


def _tc_available():
    # probe: a tiny tc GEMM either runs or reports DG_ERR_UNSUPPORTED
    lut = dg.build_lut(WL, AL, 8)
    w = gpu_pack(np.zeros((1, 4), np.uint8))
    try:
        dg.lut_gemm(w, w, 1, 1, 4, lut, variant="tc")
        return True
    except dg.DGError as e:
        if "UNSUPPORTED" in str(e):
            return False
        raise


# ---------------------------------------------------------------- pack / quantize
@pytest.mark.parametrize("K", [1, 3, 4, 63, 64, 65, 130, 576, 1001])
def test_pack_matches_oracle_unpack(K):
    g = np.random.default_rng(K)
    codes = g.integers(0, 4, (37, K), dtype=np.uint8)
    packed = gpu_pack(codes)
    assert packed.shape[1] % 16 == 0
    p = host(packed)
    assert np.array_equal(oracle.unpack_codes(p, 37, K, p.shape[1]), codes)
    # codes beyond K are zero (dg.h contract)
    full = oracle.unpack_codes(p, 37, p.shape[1] * 4, p.shape[1])
    assert not full[:, K:].any()
    # device unpack is the inverse
    assert np.array_equal(host(dg.unpack_codes(packed, K)), codes)


def test_pack_error_count():
    codes = np.array([[0, 1, 4, 3, 255, 2, 3, 1]], np.uint8)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    packed = dg.pack_codes(torch.from_numpy(codes).to(DEV), err=err)
    assert int(host(err)[0]) == 2
    assert oracle_codes_of(packed, 1, 8).tolist() == [[0, 1, 0, 3, 3, 2, 3, 1]]


@pytest.mark.parametrize("qmin,qmax", [(0, 3), (-2, 1)])
def test_quantize_pack_vs_oracle(qmin, qmax):
    g = np.random.default_rng(5)
    x = g.normal(0, 1.5, (19, 77)).astype(np.float32)
    x[0, :8] = np.array([0.25, -0.25, 0.75, -0.75, 1.25, 100, -100, 0], np.float32)  # ties, clips
    s, z = 2.0, 0.5
    packed = dg.quantize_pack_activations(torch.from_numpy(x).to(DEV), s, z, qmin, qmax)
    q = oracle.quantize(x, s, z, qmin, qmax) - qmin
    assert np.array_equal(oracle_codes_of(packed, 19, 77), q.astype(np.uint8))


# ---------------------------------------------------------------- requant
def test_requant_vs_oracle():
    g = np.random.default_rng(6)
    acc = g.integers(-5000, 5000, (33, 45)).astype(np.int32)
    res = g.integers(-300, 300, (33, 45)).astype(np.int32)
    bias = g.integers(-100, 100, 45).astype(np.int32)
    rq = dg.Requant(mult=20180, shift=20, zp=1, qmin=0, qmax=3,
                    bias=torch.from_numpy(bias).to(DEV), bias_axis=0,
                    res=torch.from_numpy(res).to(DEV))
    out = dg.requantize(torch.from_numpy(acc).to(DEV), rq)
    exp = oracle.requantize(acc, 20180, 20, 1, 0, 3, res=res, bias=bias, bias_axis=0)
    assert np.array_equal(oracle_codes_of(out, 33, 45), exp)


def test_requant_ties_exhaustive():
    acc = np.arange(-(1 << 12), 1 << 12, dtype=np.int32).reshape(-1, 64)
    for mult, shift, zp, qmin, qmax in [(1 << 19, 20, 0, -2, 1), (3, 2, 1, 0, 3), (-7, 3, 0, -1, 2)]:
        rq = dg.Requant(mult=mult, shift=shift, zp=zp, qmin=qmin, qmax=qmax)
        out = dg.requantize(torch.from_numpy(acc).to(DEV), rq)
        exp = oracle.requantize(acc, mult, shift, zp, qmin, qmax).view(np.int8).astype(np.int32) - qmin
        assert np.array_equal(oracle_codes_of(out, acc.shape[0], 64), exp.astype(np.uint8))


# ---------------------------------------------------------------- LUT GEMM
def run_gemm(W, A, lut, variant, rq=None):
    M, K = W.shape
    N = A.shape[1]
    w = gpu_pack(W, weights=True)
    at = gpu_pack(np.ascontiguousarray(A.T))
    return dg.lut_gemm(w, at, M, N, K, lut, rq=rq, variant=variant)


@pytest.mark.parametrize("variant", VARIANTS)
def test_gemm_config1(variant):
    """BJ configs[0]: M=64, N=196, K=576; int8 product table; int32 + requant codes."""
    import synth
    lut = dg.build_lut(WL, AL, 8)
    if not variant_ok(variant, lut):
        pytest.skip("tc variant unavailable")
    W = synth.uniform_codes((64, 576), 1, 0, synth.T_W)
    A = synth.uniform_codes((576, 196), 1, 0, synth.T_A)
    T = oracle.build_lut16(WL, AL)
    C = host(run_gemm(W, A, lut, variant))
    exp = oracle.lut_gemm(W, A, T)
    assert np.array_equal(C, exp)
    rq = synth.CFG1_RQ
    bias = np.full(64, rq.bias, np.int32)
    out = run_gemm(W, A, lut, variant, rq=dg.Requant(rq.mult, rq.shift, rq.zp, rq.qmin, rq.qmax,
                                                     bias=torch.from_numpy(bias).to(DEV), bias_axis=1))
    expc = oracle.requantize(exp, rq.mult, rq.shift, rq.zp, rq.qmin, rq.qmax, bias=bias, bias_axis=1)
    assert np.array_equal(oracle_codes_of(out, 64, 196), expc)


SHAPES = [(1, 1, 1), (1, 1, 4), (3, 5, 7), (64, 64, 128), (65, 63, 129), (130, 200, 300), (7, 300, 1000),
          (200, 9, 2049), (257, 129, 4608)]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_gemm_random_product(variant, M, N, K):
    lut = dg.build_lut(WL, AL, 8)
    if not variant_ok(variant, lut):
        pytest.skip("tc variant unavailable")
    g = np.random.default_rng(M * 1000 + N * 10 + K)
    W = g.integers(0, 4, (M, K), dtype=np.uint8)
    A = g.integers(0, 4, (K, N), dtype=np.uint8)
    assert np.array_equal(host(run_gemm(W, A, lut, variant)), oracle.lut_gemm(W, A, oracle.build_lut16(WL, AL)))


@pytest.mark.parametrize("seed", range(6))
def test_gemm_non_product_tables_cc(seed):
    """Arbitrary tables (LUT-16 with any precomputed entries): cc variant only."""
    g = np.random.default_rng(100 + seed)
    amp = [5, 60, 127, 1000, 16129, 1 << 20][seed]
    T = g.integers(-amp, amp + 1, 16).astype(np.int32)
    M, N, K = [(31, 17, 100), (64, 130, 257), (5, 64, 1024), (96, 40, 333), (80, 80, 2000), (33, 65, 513)][seed]
    W = g.integers(0, 4, (M, K), dtype=np.uint8)
    A = g.integers(0, 4, (K, N), dtype=np.uint8)
    lut = dg.lut_from_table(T, 32)
    exp = oracle.lut_gemm(W, A, T)
    assert np.array_equal(host(run_gemm(W, A, lut, "cc")), exp)
    assert dg.last_kernel().startswith("cc")
    with pytest.raises(dg.DGError, match="UNSUPPORTED"):
        run_gemm(W, A, lut, "tc_ss")
    if amp <= 127:   # int8 entries: the public call runs the one-hot K' = 4K tensor-core form (auto and tc)
        for v in ("auto", "tc"):
            assert np.array_equal(host(run_gemm(W, A, lut, v)), exp)
            assert dg.last_kernel().startswith("ts ")
    else:
        with pytest.raises(dg.DGError, match="UNSUPPORTED"):
            run_gemm(W, A, lut, "tc")
        assert np.array_equal(host(run_gemm(W, A, lut, "auto")), exp)   # auto falls back to the cc kernel
        assert dg.last_kernel().startswith("cc")


@pytest.mark.parametrize("variant", VARIANTS)
def test_gemm_config5_levels_small(variant):
    """Config 5 table (reading Q17: learned-style levels, int16 product table) at a small size."""
    import synth
    wl, al = synth.learned_levels(5, 0, synth.T_LEVELS)
    lut = dg.build_lut(wl, al, 16)
    if not variant_ok(variant, lut):
        pytest.skip("tc variant unavailable")
    g = np.random.default_rng(55)
    M, N, K = 160, 144, 1024
    W = g.integers(0, 4, (M, K), dtype=np.uint8)
    A = g.integers(0, 4, (K, N), dtype=np.uint8)
    assert np.array_equal(host(run_gemm(W, A, lut, variant)), oracle.lut_gemm(W, A, oracle.build_lut16(wl, al)))


def test_gemm_errors():
    lut = dg.build_lut(WL, AL, 8)
    w = gpu_pack(np.zeros((4, 8), np.uint8))
    with pytest.raises(dg.DGError, match="SHAPE"):
        dg.lut_gemm(w, w, 4, 4, 0, lut)
    with pytest.raises(dg.DGError, match="OVERFLOW"):
        dg.build_lut([127, 0, 0, 0], [127, 0, 0, 0], 8)
    big = dg.lut_from_table([1 << 30] * 16, 32)
    with pytest.raises(dg.DGError, match="OVERFLOW"):
        dg.lut_gemm(w, w, 4, 4, 8, big)


@pytest.mark.parametrize("B,H,W,C,Cout,k,stride,pad,pad_code", [
    (1, 1, 1, 64, 64, 3, 1, 1, 2),    # a 1x1 image: every tap but the centre is padding
    (3, 2, 5, 64, 128, 3, 2, 1, 1),   # stride 2 on a 2-row image
    (2, 3, 3, 256, 256, 3, 1, 0, 0),  # no padding: one output pixel per image
    (1, 1, 7, 128, 64, 1, 1, 0, 0),   # a single image row, 1x1
])
def test_conv_degenerate_images(B, H, W, C, Cout, k, stride, pad, pad_code):
    """Tiny / degenerate images through the int8 prepared conv and the FP4 conv, bit-exact."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    wl = [-2, -1, 0, 1]
    T = oracle.build_lut16(wl, AL)
    lut = dg.build_lut(wl, AL, 8)
    g = np.random.default_rng(B + H + W + C + Cout + k + pad_code)
    x = g.integers(0, 4, (B, H, W, C), dtype=np.uint8)
    w = g.integers(0, 4, (Cout, k, k, C), dtype=np.uint8)
    exp = oracle.conv2d_direct(x, w, T, stride, pad, pad_code).reshape(-1, Cout)
    xp, Cp = nhwc_pack(x)
    wp = conv_weights_pack(w, Cp)
    p = dg.conv_params(B, H, W, Cp, Cout, k, k, stride, pad, pad_code, ldw=wp.shape[1])
    ws = torch.empty(dg.conv_workspace_size(p), dtype=torch.uint8, device=DEV)
    w8 = dg.expand_operand(wp, k * k * Cp, wl)
    assert np.array_equal(host(dg.lut_conv2d_prepared(xp, w8, lut, p, ws=ws)).reshape(exp.shape), exp)
    w4 = dg.expand_operand_f4(wp, k * k * Cp, wl)
    assert np.array_equal(host(dg.lut_conv2d_f4_prepared(xp, w4, lut, p)), exp)


@pytest.mark.parametrize("variant", ["cc", "tc", "auto"])
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (1, 300, 577), (300, 1, 577), (130, 70, 1), (5, 3, 3)])
def test_gemm_degenerate_shapes(variant, M, N, K):
    """Degenerate GEMMs (a single output row / column, K = 1, K not a multiple of 4) on every
    variant: bit-exact against the oracle; all-zero activation codes (level 0) give C = 0 exactly
    (the invariant of the oracle pins), including with the fused requant."""
    lut = dg.build_lut(WL, AL, 8)
    T = oracle.build_lut16(WL, AL)
    g = np.random.default_rng(M * 31 + N * 7 + K)
    W = g.integers(0, 4, (M, K), dtype=np.uint8)
    A = g.integers(0, 4, (K, N), dtype=np.uint8)
    w, at = gpu_pack(W, weights=True), gpu_pack(np.ascontiguousarray(A.T))
    try:
        C = host(dg.lut_gemm(w, at, M, N, K, lut, variant=variant))
    except dg.DGError as e:
        assert variant == "tc" and "UNSUPPORTED" in str(e), e
        return
    assert np.array_equal(C, oracle.lut_gemm(W, A, T))
    z = gpu_pack(np.zeros((N, K), np.uint8))
    assert not host(dg.lut_gemm(w, z, M, N, K, lut, variant=variant)).any()
    rq = dg.Requant(30000, 20, 1, 0, 3)
    codes = dg.lut_gemm(w, z, M, N, K, lut, variant=variant, rq=rq)
    exp = oracle.requantize(np.zeros((M, N), np.int32), 30000, 20, 1, 0, 3)
    assert np.array_equal(oracle_codes_of(codes, M, N), exp)


# ---------------------------------------------------------------- conv
def nhwc_pack(x):
    B, H, W, C = x.shape
    Cp = (C + 3) // 4 * 4
    xc = np.zeros((B * H * W, Cp), np.uint8)
    xc[:, :C] = x.reshape(-1, C)
    # pack rows of Cp codes into exactly Cp/4 bytes (NHWC packed), via the GPU packer
    p = gpu_pack(xc)
    return p[:, :Cp // 4].contiguous(), Cp


def conv_weights_pack(w, Cp, wpad=2):
    Cout, kh, kw, C = w.shape
    wc = np.full((Cout, kh, kw, Cp), wpad, np.uint8)
    wc[..., :C] = w
    return gpu_pack(wc.reshape(Cout, -1), weights=True)


CONVS = [  # B, H, W, C, Cout, k, stride, pad, pad_code
    (1, 8, 8, 16, 16, 3, 1, 1, 0),
    (2, 9, 7, 12, 20, 3, 2, 1, 0),
    (2, 6, 6, 64, 32, 1, 1, 0, 0),     # direct (no im2col) path
    (2, 7, 7, 64, 64, 1, 2, 0, 0),     # strided 1x1 (downsample)
    (1, 10, 10, 3, 16, 3, 1, 1, 0),    # VGG conv1_1-like, Cin=3 padded to 4
    (1, 5, 5, 8, 8, 3, 1, 1, 2),       # non-zero pad code
    (3, 14, 14, 128, 64, 3, 1, 1, 0),
    (2, 9, 9, 64, 32, 3, 1, 1, 2),     # implicit-GEMM path with a non-zero pad code
    (1, 12, 12, 256, 64, 3, 2, 1, 0),  # implicit, stride 2, C/4 = 64
    (2, 10, 10, 64, 64, 1, 2, 0, 0),   # implicit 1x1 stride 2 (downsample)
    (1, 11, 13, 64, 32, 5, 2, 2, 1),   # implicit 5x5 (25 taps: precomputed tap masks), pad 2, pad code 1
    (1, 9, 9, 64, 16, 7, 1, 3, 0),     # implicit 7x7 (49 taps > 32: per-chunk tap arithmetic)
]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("B,H,W,C,Cout,k,stride,pad,pad_code", CONVS)
def test_conv_vs_oracle(variant, B, H, W, C, Cout, k, stride, pad, pad_code):
    lut = dg.build_lut(WL, AL, 8)
    if not variant_ok(variant, lut):
        pytest.skip("tc variant unavailable")
    g = np.random.default_rng(B * 7 + H + C + Cout + k)
    x = g.integers(0, 4, (B, H, W, C), dtype=np.uint8)
    w = g.integers(0, 4, (Cout, k, k, C), dtype=np.uint8)
    T = oracle.build_lut16(WL, AL)
    exp = oracle.conv2d_direct(x, w, T, stride, pad, pad_code)
    xp, Cp = nhwc_pack(x)
    wp = conv_weights_pack(w, Cp)
    p = dg.conv_params(B, H, W, Cp, Cout, k, k, stride, pad, pad_code, ldw=wp.shape[1])
    try:
        out = dg.lut_conv2d(xp, wp, lut, p, variant=variant)
    except dg.DGError as e:
        if variant.startswith("tc") and pad_code != 0 and "UNSUPPORTED" in str(e):
            pytest.skip("tc conv requires pad level 0")
        raise
    assert np.array_equal(host(out).reshape(exp.shape), exp)
    # fused requant with a per-channel bias
    bias = g.integers(-50, 50, Cout).astype(np.int32)
    rq = dg.Requant(mult=30000, shift=20, zp=1, bias=torch.from_numpy(bias).to(DEV), bias_axis=0)
    outc = dg.lut_conv2d(xp, wp, lut, p, rq=rq, variant=variant)
    expc = oracle.requantize(exp.reshape(-1, Cout), 30000, 20, 1, 0, 3, bias=bias, bias_axis=0)
    assert np.array_equal(oracle_codes_of(outc, expc.shape[0], Cout), expc)


@pytest.mark.parametrize("variant", VARIANTS)
def test_conv_residual_identity_and_downsample(variant):
    """O-RES (reading Q13): identity shortcut r = al[x]*res_mult over packed codes, and a
    downsample shortcut r = int32 accumulator of a 1x1 stride-2 conv."""
    lut = dg.build_lut(WL, AL, 8)
    if not variant_ok(variant, lut):
        pytest.skip("tc variant unavailable")
    g = np.random.default_rng(77)
    T = oracle.build_lut16(WL, AL)
    B, H, C = 2, 8, 64
    x = g.integers(0, 4, (B, H, H, C), dtype=np.uint8)
    w = g.integers(0, 4, (C, 3, 3, C), dtype=np.uint8)
    xp, Cp = nhwc_pack(x)
    wp = conv_weights_pack(w, Cp)
    p = dg.conv_params(B, H, H, C, C, 3, 3, 1, 1, 0, ldw=wp.shape[1])
    acc = oracle.conv2d_direct(x, w, T, 1, 1, 0).reshape(-1, C)
    res_mult = 37
    rq = dg.Requant(mult=15000, shift=20, zp=0, res_codes=xp, res_mult=res_mult, res_levels=AL)
    out = dg.lut_conv2d(xp, wp, lut, p, rq=rq, variant=variant)
    r = (np.array(AL)[x.reshape(-1, C)] * res_mult).astype(np.int32)
    exp = oracle.requantize(acc, 15000, 20, 0, 0, 3, res=r)
    assert np.array_equal(oracle_codes_of(out, exp.shape[0], C), exp)
    # downsample: 1x1 stride 2 conv accumulators as the residual of a stride-2 3x3 conv
    C2 = 128
    w2 = g.integers(0, 4, (C2, 3, 3, C), dtype=np.uint8)
    wd = g.integers(0, 4, (C2, 1, 1, C), dtype=np.uint8)
    w2p, wdp = conv_weights_pack(w2, Cp), conv_weights_pack(wd, Cp)
    pd = dg.conv_params(B, H, H, C, C2, 1, 1, 2, 0, 0, ldw=wdp.shape[1])
    p2 = dg.conv_params(B, H, H, C, C2, 3, 3, 2, 1, 0, ldw=w2p.shape[1])
    racc = dg.lut_conv2d(xp, wdp, lut, pd, variant=variant)
    out2 = dg.lut_conv2d(xp, w2p, lut, p2, rq=dg.Requant(mult=12000, shift=20, res=racc), variant=variant)
    a2 = oracle.conv2d_direct(x, w2, T, 2, 1, 0).reshape(-1, C2)
    rd = oracle.conv2d_direct(x, wd, T, 2, 0, 0).reshape(-1, C2)
    assert np.array_equal(host(racc), rd)
    exp2 = oracle.requantize(a2, 12000, 20, 0, 0, 3, res=rd)
    assert np.array_equal(oracle_codes_of(out2, exp2.shape[0], C2), exp2)


@pytest.mark.parametrize("M,N,K", [(130, 70, 300), (256, 256, 1024), (77, 129, 64), (128, 64, 4608)])
def test_gemm_prepared_and_expand(M, N, K):
    """dg_expand_operand + dg_lut_gemm_prepared (offline-expanded second operand) vs the oracle;
    the expansion itself is checked against the levels (zero beyond K) up to the documented order."""
    import synth
    wl, al = synth.learned_levels(5, 1, synth.T_LEVELS)
    lut = dg.build_lut(wl, al, 16)
    if not _tc_available():
        pytest.skip("tc unavailable")
    g = np.random.default_rng(M + N + K)
    W = g.integers(0, 4, (M, K), dtype=np.uint8)
    A = g.integers(0, 4, (K, N), dtype=np.uint8)
    w = gpu_pack(W, weights=True)
    at = gpu_pack(np.ascontiguousarray(A.T))
    at8 = dg.expand_operand(at, K, al)
    e = host(at8).astype(np.int64)
    assert e.shape[1] % 128 == 0 and not e[:, K + (-K) % 16:].any()
    # per 16-code word the multiset of levels is preserved (order: 0,2,..,14,1,3,..,15)
    perm = [0, 2, 4, 6, 8, 10, 12, 14, 1, 3, 5, 7, 9, 11, 13, 15]
    Kw = K // 16 * 16
    lv = np.array(al, np.int64)[A.T[:, :Kw]].reshape(N, -1, 16)[:, :, perm]
    assert np.array_equal(e[:, :Kw].reshape(N, -1, 16), lv)
    C = host(dg.lut_gemm_prepared(w, at8, M, N, K, lut))
    assert np.array_equal(C, oracle.lut_gemm(W, A, oracle.build_lut16(wl, al)))


@pytest.mark.parametrize("P,m,N,K", [(3, 200, 300, 576), (2, 128, 64, 4608), (8, 40, 130, 100)])
def test_gemm_fused_allgather(P, m, N, K):
    """dg_lut_gemm_prepared_allgather: P simulated ranks on one GPU, each computing its m-row block
    and storing it into all P full-C buffers (its own + P-1 'peer' destinations at its row
    offset).  Every buffer must end up equal to the oracle's full C (config 5's exchange step)."""
    import synth
    if not _tc_available():
        pytest.skip("tc unavailable")
    wl, al = synth.learned_levels(5, 2, synth.T_LEVELS)
    lut = dg.build_lut(wl, al, 16)
    g = np.random.default_rng(P * 1000 + m + N + K)
    M = P * m
    W = g.integers(0, 4, (M, K), dtype=np.uint8)
    A = g.integers(0, 4, (K, N), dtype=np.uint8)
    at8 = dg.expand_operand(gpu_pack(np.ascontiguousarray(A.T)), K, al)
    full = [torch.full((M, N), -7, dtype=torch.int32, device=DEV) for _ in range(P)]
    n0 = dg.kernel_launches()
    for r in range(P):
        w_r = gpu_pack(np.ascontiguousarray(W[r * m:(r + 1) * m]), weights=True)
        peers = [full[j][r * m:].data_ptr() for j in range(P) if j != r]
        n1 = dg.kernel_launches()
        dg.lut_gemm_prepared_allgather(w_r, at8, m, N, K, lut, full[r][r * m:(r + 1) * m], peers)
        assert dg.kernel_launches() - n1 == 1   # one fused kernel per rank, no separate collective
    exp = oracle.lut_gemm(W, A, oracle.build_lut16(wl, al))
    for j in range(P):
        assert np.array_equal(host(full[j]), exp), j
    with pytest.raises(dg.DGError, match="UNSUPPORTED"):
        dg.lut_gemm_prepared_allgather(w_r, at8, m, N, K, lut, full[0][:m], [full[0].data_ptr()] * 8)


@pytest.mark.parametrize("B,H,W,C,Cout,k,stride,pad,pad_code", CONVS)
def test_conv_prepared_vs_oracle(B, H, W, C, Cout, k, stride, pad, pad_code):
    """dg_lut_conv2d_prepared (offline-expanded weights; direct / implicit-GEMM / im2col)."""
    lut = dg.build_lut(WL, AL, 8)
    if not _tc_available():
        pytest.skip("tc unavailable")
    g = np.random.default_rng(B * 11 + H + C + Cout + k + pad_code)
    x = g.integers(0, 4, (B, H, W, C), dtype=np.uint8)
    w = g.integers(0, 4, (Cout, k, k, C), dtype=np.uint8)
    exp = oracle.conv2d_direct(x, w, oracle.build_lut16(WL, AL), stride, pad, pad_code)
    xp, Cp = nhwc_pack(x)
    wp = conv_weights_pack(w, Cp)
    Kc = k * k * Cp
    w8 = dg.expand_operand(wp, Kc, WL)
    p = dg.conv_params(B, H, W, Cp, Cout, k, k, stride, pad, pad_code, ldw=wp.shape[1])
    ws = torch.empty(dg.conv_workspace_size(p), dtype=torch.uint8, device=DEV)
    out = dg.lut_conv2d_prepared(xp, w8, lut, p, ws=ws)
    assert np.array_equal(host(out).reshape(exp.shape), exp)


# ---------------------------------------------------------------- requant epilogue paths
RQ_SWEEP = [  # mult, zp, qmin, qmax, bias kind
    (30000, 0, 0, 3, "none"),
    (30000, 1, 0, 3, "col"),          # per-column bias table (16-bit SIMD path)
    (5000, 0, 0, 3, "col"),           # wide threshold spacing
    (200000, 2, 0, 3, "uniform"),     # narrow spacing (~5 accumulator units)
    (1 << 20, 1, 0, 3, "col"),        # spacing exactly 1: consecutive thresholds
    (3 << 20, 0, 0, 3, "none"),       # spacing < 1: some codes unreachable / equal thresholds
    (20180, 1, -1, 2, "col"),         # signed code range (qmin = -1)
    (30000, 0, 0, 2, "col"),          # only 3 codes used (an infinite threshold)
    (-30000, 0, 0, 3, "col"),         # negative multiplier (decreasing map)
    (30000, 0, 0, 3, "colbig"),       # |bias| near 2^15: 16-bit offsets overflow -> 32-bit path
    (30000, 1, 0, 3, "row"),          # GEMM orientation: bias per row (TMEM lane)
]


@pytest.mark.parametrize("mult,zp,qmin,qmax,bias_kind", RQ_SWEEP)
@pytest.mark.parametrize("K", [64, 2304])
def test_tc_requant_epilogue_sweep(mult, zp, qmin, qmax, bias_kind, K):
    """Fused requant on the tensor-core path (16-bit SIMD epilogue where its host-verified
    parameters exist, else the 32-bit threshold path) against O-REQ over the oracle's
    accumulators, bit-exact, for spacings, signed ranges, unreachable codes, bias layouts
    and offsets that overflow 16 bits."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    lut = dg.build_lut(WL, AL, 8)
    T = oracle.build_lut16(WL, AL)
    g = np.random.default_rng(K + abs(mult) % 1000 + zp + qmin)
    M, N = 300, 96                      # M = pixels (TMEM lanes, ragged last tile), N = channels
    A = g.integers(0, 4, (M, K), dtype=np.uint8)       # activations, K-major
    Wt = g.integers(0, 4, (N, K), dtype=np.uint8)      # weights [channel][K]
    acc = oracle.lut_gemm(A, np.ascontiguousarray(Wt.T), oracle.build_lut16(AL, WL))   # [M][N]
    assert np.array_equal(acc, oracle.lut_gemm(Wt, np.ascontiguousarray(A.T), T).T)
    mu = int(np.round(acc.mean()))
    if bias_kind == "none":
        bias, axis = None, 0
    elif bias_kind == "uniform":
        bias, axis = np.full(N, -mu, np.int32), 0
    elif bias_kind == "col":
        bias, axis = (-mu + g.integers(-40, 40, N)).astype(np.int32), 0
    elif bias_kind == "colbig":
        bias, axis = (-mu + g.integers(-40, 40, N)).astype(np.int32), 0
        bias[5] = 32000
    else:
        bias, axis = (-mu + g.integers(-40, 40, M)).astype(np.int32), 1
    a_p = gpu_pack(A)
    w_p = gpu_pack(Wt, weights=True)
    w8 = dg.expand_operand(w_p, K, WL)
    lut_t = dg.build_lut(AL, WL, 8)   # index (a<<2)|w: P = activations
    rq = dg.Requant(mult, 20, zp, qmin, qmax, bias=None if bias is None else torch.from_numpy(bias).to(DEV),
                    bias_axis=axis)
    got = dg.lut_gemm_prepared(a_p, w8, M, N, K, lut_t, rq=rq)
    q = oracle.requantize(acc, mult, 20, zp, qmin, qmax, bias=bias, bias_axis=axis).view(np.int8)
    exp = (q.astype(np.int32) - qmin).astype(np.uint8)     # dg.h: code = q - qmin
    assert np.array_equal(oracle_codes_of(got, M, N), exp)


WIN_CONVS = [  # B, H, W, C, Cout, pad_code: 3x3 / stride 1 / pad 1 shapes of the shifted-window path
    (2, 9, 9, 64, 32, 0),
    (3, 14, 14, 128, 64, 0),
    (1, 7, 11, 256, 128, 2),      # non-square, non-zero pad code
    (2, 56, 56, 64, 64, 0),       # ResNet-50 stage-1 width (window of 248 rows)
    (2, 12, 10, 64, 128, 0),      # C = 64 tile mode with 128-wide tiles (VGG conv2_1 shape class)
    (1, 23, 17, 64, 64, 3),       # C = 64 tile mode, ragged last tile, pad code 3
    (1, 10, 120, 64, 64, 0),      # wide: 374-row window, 2 rows per unpack thread
    (1, 6, 224, 64, 128, 1),      # VGG width: 582-row window, 3 rows per thread, pad code 1
    (3, 28, 28, 128, 128, 0),     # C = 128 tile mode (weights resident), ResNet-50 stage-2 shape
    (2, 20, 13, 128, 96, 2),      # C = 128 tile mode, ragged Cout and tiles, pad code 2
    (1, 9, 112, 128, 128, 0),     # C = 128 at VGG width: one window (2 rows per thread) beside the weights
]


def _win_check(B, H, W, C, Cout, pad_code, expect, exact_images=None):
    """Window-kernel conv vs the oracle: int32 output (element by element) and fused requant with a
    per-channel bias; asserts that the instance which ran carries every tag in `expect`."""
    lut = dg.build_lut(WL, AL, 8)
    g = np.random.default_rng(B + H + W + C + Cout + pad_code)
    x = g.integers(0, 4, (B, H, W, C), dtype=np.uint8)
    w = g.integers(0, 4, (Cout, 3, 3, C), dtype=np.uint8)
    exp = oracle.conv2d_direct(x, w, oracle.build_lut16(WL, AL), 1, 1, pad_code)
    xp, Cp = nhwc_pack(x)
    wp = conv_weights_pack(w, Cp)
    w8 = dg.expand_operand(wp, 9 * Cp, WL)
    p = dg.conv_params(B, H, W, Cp, Cout, 3, 3, 1, 1, pad_code, ldw=wp.shape[1])
    ws = torch.empty(dg.conv_workspace_size(p), dtype=torch.uint8, device=DEV)
    out = dg.lut_conv2d_prepared(xp, w8, lut, p, ws=ws)
    tag = dg.last_kernel()
    for e in expect:
        assert e in tag, (e, tag)
    assert np.array_equal(host(out).reshape(exp.shape), exp)
    bias = g.integers(-50, 50, Cout).astype(np.int32)
    rq = dg.Requant(mult=30000, shift=20, zp=1, bias=torch.from_numpy(bias).to(DEV), bias_axis=0)
    outc = dg.lut_conv2d_prepared(xp, w8, lut, p, rq=rq, ws=ws)
    assert dg.last_kernel().split(" f16=")[0] == tag.split(" f16=")[0]   # same instance (f16: requant only)
    expc = oracle.requantize(exp.reshape(-1, Cout), 30000, 20, 1, 0, 3, bias=bias, bias_axis=0)
    assert np.array_equal(oracle_codes_of(outc, expc.shape[0], Cout), expc)


@pytest.mark.parametrize("B,H,W,C,Cout,pad_code,win128",
                         [c + (0,) for c in WIN_CONVS] +
                         [c + (1,) for c in WIN_CONVS if c[3] == 128 and c[4] <= 128])
def test_conv_window_path_vs_oracle(win128, B, H, W, C, Cout, pad_code):
    """Direct 3x3 conv through the shifted-window kernel, FORCED (dg_set_option win=1) on shapes
    below its two-wave auto threshold: one unpacked window of padded input pixels per tile, every
    tap an MMA on a row-shifted shared-memory descriptor, vs O-CONV, int32 and fused requant.
    C = 128 / Cout <= 128 runs the C = 128 tile mode (win128=1) or the 256-code stage form."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    expect = [" win "] + (["kst=128"] if win128 else ["kst=256"])
    with dg.options(win=1, win128=win128):
        _win_check(B, H, W, C, Cout, pad_code, expect)


DEFAULT_WIN = [  # shapes that select each default window instance with NO option forced (>= 2 waves)
    (48, 28, 28, 128, 128, 0, ["kst=128", "nwin=2"]),           # C = 128 tile mode, 2 windows (R-50 stage 2)
    (3, 112, 112, 128, 128, 2, ["kst=128", "nwin=1"]),          # C = 128 at 112 wide: 1 window (VGG conv2_2)
    (3, 112, 112, 64, 128, 0, ["bn=128", "kst=256", "wpair=1"]),   # 64 -> 128 pair mode (VGG conv2_1)
    (12, 56, 56, 64, 64, 1, ["bn=64", "kst=256", "wpair=1"]),      # 64 -> 64 pair mode (R-50 stage 1)
    (2, 224, 224, 64, 64, 0, ["bn=64", "wpair=1"]),              # VGG width: 3 window rows per thread
]


@pytest.mark.parametrize("B,H,W,C,Cout,pad_code,expect", DEFAULT_WIN)
def test_conv_window_default_instances_vs_oracle(B, H, W, C, Cout, pad_code, expect):
    """Every window instance the auto dispatch picks for the bench's layers, at a size that picks it
    by default (checked through dg_last_kernel), bit-exact against the oracle's direct conv."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    dg.reset_options()
    _win_check(B, H, W, C, Cout, pad_code, [" win "] + expect)


@pytest.mark.parametrize("C2,res_mult", [(64, 37), (128, 900), (64, 20000)])
def test_conv_residual_16bit_path(C2, res_mult):
    """Residual requant (reading Q13) through the tensor-core 16-bit epilogue: identity shortcut
    over packed codes (pair table) and int32 downsample shortcut (|r| < 2^14 fast, else exact
    redo); res_mult 20000 exceeds the 16-bit range and must take the exact path."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    lut = dg.build_lut(WL, AL, 8)
    T = oracle.build_lut16(WL, AL)
    g = np.random.default_rng(C2 + res_mult)
    B, H, C = 2, 10, 64
    x = g.integers(0, 4, (B, H, H, C), dtype=np.uint8)
    w = g.integers(0, 4, (C, 3, 3, C), dtype=np.uint8)
    xp, Cp = nhwc_pack(x)
    wp = conv_weights_pack(w, Cp)
    w8 = dg.expand_operand(wp, 9 * Cp, WL)
    p = dg.conv_params(B, H, H, C, C, 3, 3, 1, 1, 0, ldw=wp.shape[1])
    ws = torch.empty(dg.conv_workspace_size(p), dtype=torch.uint8, device=DEV)
    acc = oracle.conv2d_direct(x, w, T, 1, 1, 0).reshape(-1, C)
    bias = g.integers(-60, 60, C).astype(np.int32)
    rq = dg.Requant(mult=15000, shift=20, zp=0, bias=torch.from_numpy(bias).to(DEV), bias_axis=0,
                    res_codes=xp, res_mult=res_mult, res_levels=AL)
    out = dg.lut_conv2d_prepared(xp, w8, lut, p, rq=rq, ws=ws)
    r = (np.array(AL)[x.reshape(-1, C)] * res_mult).astype(np.int32)
    exp = oracle.requantize(acc, 15000, 20, 0, 0, 3, res=r, bias=bias, bias_axis=0)
    assert np.array_equal(oracle_codes_of(out, exp.shape[0], C), exp)
    # int32 residual: a 1x1 stride-2 downsample's accumulators, scaled to reach the 2^14 limit
    w2 = g.integers(0, 4, (C2, 3, 3, C), dtype=np.uint8)
    wd = g.integers(0, 4, (C2, 1, 1, C), dtype=np.uint8)
    w2p, wdp = conv_weights_pack(w2, Cp), conv_weights_pack(wd, Cp)
    w28, wd8 = dg.expand_operand(w2p, 9 * Cp, WL), dg.expand_operand(wdp, Cp, WL)
    pd = dg.conv_params(B, H, H, C, C2, 1, 1, 2, 0, 0, ldw=wdp.shape[1])
    p2 = dg.conv_params(B, H, H, C, C2, 3, 3, 2, 1, 0, ldw=w2p.shape[1])
    racc = dg.lut_conv2d_prepared(xp, wd8, lut, pd, ws=ws)
    rd = oracle.conv2d_direct(x, wd, T, 2, 0, 0).reshape(-1, C2)
    assert np.array_equal(host(racc), rd)
    scale = max(1, res_mult // 100)
    racc_s = (racc * scale).contiguous()
    out2 = dg.lut_conv2d_prepared(xp, w28, lut, p2, rq=dg.Requant(mult=12000, shift=20, res=racc_s), ws=ws)
    a2 = oracle.conv2d_direct(x, w2, T, 2, 1, 0).reshape(-1, C2)
    exp2 = oracle.requantize(a2, 12000, 20, 0, 0, 3, res=(rd * scale).astype(np.int32))
    assert np.array_equal(oracle_codes_of(out2, exp2.shape[0], C2), exp2)


SPLITK_CONVS = [  # B, H, C, Cout, k, stride: few output tiles, long K -> split-K partial sums
    (1, 14, 256, 256, 3, 1),
    (1, 7, 512, 512, 3, 1),
    (1, 14, 256, 512, 1, 2),
    (2, 7, 128, 64, 3, 1),
    (1, 7, 256, 70, 3, 1),        # ragged Cout (int32 output only)
]


@pytest.mark.parametrize("skfuse", [1, 0])
@pytest.mark.parametrize("B,H,C,Cout,k,stride", SPLITK_CONVS)
def test_conv_splitk_vs_oracle(B, H, C, Cout, k, stride, skfuse):
    """Small-batch convs (ResNet-18 b1 shapes) whose few output tiles run as split-K: each split
    writes its int32 partial slice into the workspace tail (garbage on entry); the slices are summed
    and requantised by the GEMM kernel itself after a grid-wide barrier (cooperative launch,
    skfuse = 1, one launch) or by the reduce kernel (skfuse = 0, two launches); int32 output, fused
    requant and an int32 residual."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    dg.reset_options()
    dg.set_option("skfuse", skfuse)
    lut = dg.build_lut(WL, AL, 8)
    T = oracle.build_lut16(WL, AL)
    g = np.random.default_rng(B * 100 + H + C + Cout + k)
    pad = k // 2
    x = g.integers(0, 4, (B, H, H, C), dtype=np.uint8)
    w = g.integers(0, 4, (Cout, k, k, C), dtype=np.uint8)
    exp = oracle.conv2d_direct(x, w, T, stride, pad, 0)
    xp, Cp = nhwc_pack(x)
    wp = conv_weights_pack(w, Cp)
    w8 = dg.expand_operand(wp, k * k * Cp, WL)
    p = dg.conv_params(B, H, H, Cp, Cout, k, k, stride, pad, 0, ldw=wp.shape[1])
    ws = torch.full((dg.conv_workspace_size(p),), 0xA5, dtype=torch.uint8, device=DEV)
    n0 = dg.kernel_launches()
    out = dg.lut_conv2d_prepared(xp, w8, lut, p, ws=ws)
    if k == 3:   # implicit GEMM split over K (+ the reduce kernel)
        assert dg.kernel_launches() - n0 == (1 if skfuse else 2)
        assert "skinst" in dg.last_kernel() and "sk=1 " not in dg.last_kernel(), dg.last_kernel()
        assert (" fused " in dg.last_kernel()) == bool(skfuse), dg.last_kernel()
    assert np.array_equal(host(out).reshape(exp.shape), exp)
    if Cout % 4:
        return
    bias = g.integers(-50, 50, Cout).astype(np.int32)
    rq = dg.Requant(mult=30000, shift=20, zp=1, bias=torch.from_numpy(bias).to(DEV), bias_axis=0)
    outc = dg.lut_conv2d_prepared(xp, w8, lut, p, rq=rq, ws=ws)
    e2 = exp.reshape(-1, Cout)
    expc = oracle.requantize(e2, 30000, 20, 1, 0, 3, bias=bias, bias_axis=0)
    assert np.array_equal(oracle_codes_of(outc, expc.shape[0], Cout), expc)
    res = g.integers(-3000, 3000, e2.shape).astype(np.int32)
    outr = dg.lut_conv2d_prepared(xp, w8, lut, p, rq=dg.Requant(mult=20000, shift=20, res=torch.from_numpy(res).to(DEV)), ws=ws)
    expr = oracle.requantize(e2, 20000, 20, 0, 0, 3, res=res)
    assert np.array_equal(oracle_codes_of(outr, expr.shape[0], Cout), expr)
    dg.reset_options()


# ---- block-scaled FP4 path (tcgen05 kind::mxf4) -------------------------
F4_SHAPES = [(256, 128, 256), (300, 200, 576), (64, 196, 576), (513, 129, 1000), (256, 384, 4608), (40, 7, 3)]


@pytest.mark.parametrize("M,N,K", F4_SHAPES)
def test_gemm_f4_vs_oracle(M, N, K):
    """dg_expand_operand_f4 + dg_lut_gemm_f4 vs the oracle, bit-exact: ragged M / N / K (K not a
    multiple of the 64-code MMA step or of the 256-code stage), several tiles, config-1 levels."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    lut = dg.build_lut(WL, AL, 8)
    g = np.random.default_rng(7 * M + N + K)
    W = g.integers(0, 4, (M, K), dtype=np.uint8)
    A = g.integers(0, 4, (K, N), dtype=np.uint8)
    w4 = dg.expand_operand_f4(gpu_pack(W, weights=True), K, WL)
    C = host(dg.lut_gemm_f4(w4, gpu_pack(np.ascontiguousarray(A.T)), M, N, K, lut))
    assert np.array_equal(C, oracle.lut_gemm(W, A, oracle.build_lut16(WL, AL)))


@pytest.mark.parametrize("wl", [(-2, -1, 0, 1), (-12, -3, 4, 8), (0, 6, -6, 1), (3, 3, -2, 2)])
def test_gemm_f4_levels_and_extremes(wl):
    """Every e2m1-representable weight level set (v/2 in e2m1) at the LARGEST K the API admits
    (K * max|entry| just below 2^22, api.cu) in the adversarial order for an fp32 accumulator that
    might truncate: half the rows / columns carry the max-magnitude product on every k < K - 64
    (|partial sum| climbing to ~2^22), then 64 random small terms that must still land exactly;
    the other half random.  Bit-exact against the oracle."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    lut = dg.build_lut(list(wl), AL, 8)
    T = oracle.build_lut16(list(wl), AL)
    M, N = 48, 40
    K = ((1 << 22) - 1) // int(np.abs(T).max())
    g = np.random.default_rng(sum(wl) + 100)
    W = g.integers(0, 4, (M, K), dtype=np.uint8)
    A = g.integers(0, 4, (K, N), dtype=np.uint8)
    big_w = int(np.argmax(np.abs(np.array(wl))))
    W[::2, : K - 64] = big_w          # half the rows: max |level| first, random tail
    A[: K - 64, ::2] = 3
    w4 = dg.expand_operand_f4(gpu_pack(W, weights=True), K, list(wl))
    C = host(dg.lut_gemm_f4(w4, gpu_pack(np.ascontiguousarray(A.T)), M, N, K, lut))
    exp = oracle.lut_gemm(W, A, T)
    assert np.abs(exp).max() >= (1 << 21) + (1 << 20)   # the admitted bound is really reached
    assert np.array_equal(C, exp)
    with pytest.raises(dg.DGError, match="OVERFLOW"):   # one more code and the API refuses
        dg.lut_gemm_f4(dg.expand_operand_f4(gpu_pack(W[:8, :1].repeat(K + 1, 1), weights=True), K + 1, list(wl)),
                       gpu_pack(np.zeros((8, K + 1), np.uint8)), 8, 8, K + 1, lut)


def test_gemm_f4_rejects():
    """Tables outside the FP4 path's exact domain are refused, not approximated."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    K, M, N = 64, 8, 8
    w = gpu_pack(np.zeros((M, K), np.uint8), weights=True)
    at = gpu_pack(np.zeros((N, K), np.uint8))
    with pytest.raises(dg.DGError, match="UNSUPPORTED"):
        dg.expand_operand_f4(w, K, [-5, -1, 0, 1])          # 5/2 is not an e2m1 value
    w4 = dg.expand_operand_f4(w, K, WL)
    with pytest.raises(dg.DGError, match="UNSUPPORTED"):   # activation levels must be 0..3
        dg.lut_gemm_f4(w4, at, M, N, K, dg.build_lut(WL, [0, 1, 2, 4], 8))
    with pytest.raises(dg.DGError, match="OVERFLOW"):      # K * 12 * 3 >= 2^22
        big = 120000
        wb = gpu_pack(np.zeros((M, big), np.uint8), weights=True)
        ab = gpu_pack(np.zeros((N, big), np.uint8))
        dg.lut_gemm_f4(dg.expand_operand_f4(wb, big, [-12, 0, 1, 2]), ab, M, N, big,
                       dg.build_lut([-12, 0, 1, 2], AL, 8))


# ---- non-product tables on the tensor cores (one-hot K' = 4K form) ----------
@pytest.mark.parametrize("seed", range(6))
def test_gemm_onehot_non_product_vs_oracle(seed):
    """Arbitrary int8 tables (not wl x al): dg_expand_onehot + dg_expand_tcols + dg_lut_gemm_onehot
    equal the oracle's direct lookup sum bit for bit, ragged M / N / K, several tiles."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    g = np.random.default_rng(300 + seed)
    amp = [1, 5, 60, 127, 127, 100][seed]
    T = g.integers(-amp, amp + 1, 16).astype(np.int32)
    M, N, K = [(31, 17, 100), (64, 130, 257), (300, 200, 576), (96, 40, 333), (256, 384, 2000), (129, 65, 7)][seed]
    W = g.integers(0, 4, (M, K), dtype=np.uint8)
    A = g.integers(0, 4, (K, N), dtype=np.uint8)
    lut = dg.lut_from_table(T, 8)
    w1h = dg.expand_onehot(gpu_pack(W, weights=True), K)
    atc = dg.expand_tcols(gpu_pack(np.ascontiguousarray(A.T)), K, lut)
    C = host(dg.lut_gemm_onehot(w1h, atc, M, N, K, lut))
    assert np.array_equal(C, oracle.lut_gemm(W, A, T))


@pytest.mark.parametrize("B,H,W,C,Cout,k,stride,pad,pad_code", [(2, 9, 7, 64, 32, 3, 1, 1, 2), (1, 10, 10, 12, 20, 3, 2, 1, 1),
                                                                   (2, 6, 6, 64, 64, 1, 1, 0, 0), (1, 9, 9, 8, 16, 5, 1, 2, 3)])
def test_conv_non_product_table_public_call(B, H, W, C, Cout, k, stride, pad, pad_code):
    """dg_lut_conv2d with a NON-product int8 table (any 16 entries): im2col + one-hot
    activations + weight table columns on the tensor cores, int32 and fused requant, vs O-CONV."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    g = np.random.default_rng(B + H + C + Cout + k + pad_code)
    T = g.integers(-127, 128, 16).astype(np.int32)
    lut = dg.lut_from_table(T, 8)
    x = g.integers(0, 4, (B, H, W, C), dtype=np.uint8)
    w = g.integers(0, 4, (Cout, k, k, C), dtype=np.uint8)
    exp = oracle.conv2d_direct(x, w, T, stride, pad, pad_code)
    xp, Cp = nhwc_pack(x)
    wp = conv_weights_pack(w, Cp, wpad=0)
    if Cp != C:   # padded channels must contribute nothing: pad weights and activations with codes whose entry is 0
        pytest.skip("non-product tables need C % 4 == 0 (no neutral pad code in general)")
    p = dg.conv_params(B, H, W, Cp, Cout, k, k, stride, pad, pad_code, ldw=wp.shape[1])
    out = dg.lut_conv2d(xp, wp, lut, p)
    assert dg.last_kernel().startswith("ts "), dg.last_kernel()
    assert np.array_equal(host(out).reshape(exp.shape), exp)
    mu = int(np.round(exp.mean()))
    rq = dg.Requant(mult=15000, shift=20, zp=1, bias=torch.full((Cout,), -mu, dtype=torch.int32, device=DEV))
    outc = dg.lut_conv2d(xp, wp, lut, p, rq=rq)
    expc = oracle.requantize(exp.reshape(-1, Cout), 15000, 20, 1, 0, 3, bias=np.full(Cout, -mu, np.int32), bias_axis=0)
    assert np.array_equal(oracle_codes_of(outc, expc.shape[0], Cout), expc)


def test_gemm_onehot_operands_and_requant():
    """The one-hot operand is 1 << (2 * code) per original code (documented packed format); the fused
    requant epilogue on the K' = 4K path equals the oracle's requantised codes; >127 entries refused."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    g = np.random.default_rng(77)
    T = g.integers(-100, 101, 16).astype(np.int32)
    M, N, K = 128, 256, 576
    W = g.integers(0, 4, (M, K), dtype=np.uint8)
    A = g.integers(0, 4, (K, N), dtype=np.uint8)
    lut = dg.lut_from_table(T, 8)
    w1h = host(dg.expand_onehot(gpu_pack(W, weights=True), K))
    assert np.array_equal(w1h[:, :K], (1 << (2 * W.astype(np.int32))).astype(np.uint8))
    assert not w1h[:, K:].any()
    exp = oracle.lut_gemm(W, A, T)
    rq = dg.Requant(20180, 20, 1, 0, 3)
    codes = dg.lut_gemm_onehot(torch.from_numpy(w1h).to(DEV), dg.expand_tcols(gpu_pack(np.ascontiguousarray(A.T)), K, lut),
                               M, N, K, lut, rq=rq)
    got = oracle.unpack_codes(host(codes), M, N, codes.shape[1])
    assert np.array_equal(got, oracle.requantize(exp, 20180, 20, 1, 0, 3))
    big = dg.lut_from_table(np.full(16, 200, np.int32), 16)
    with pytest.raises(dg.DGError, match="UNSUPPORTED"):
        dg.expand_tcols(gpu_pack(np.ascontiguousarray(A.T)), K, big)


# ---- 4-bit operands as 2-bit digit pairs (Table 2) --------------
def _levels16(seed, amp=31):
    return np.random.default_rng(seed).integers(-amp, amp + 1, 16).astype(np.int32)


@pytest.mark.parametrize("B,H,W,C,k,stride,pad,pad_code", [
    (2, 9, 11, 4, 3, 1, 1, 0),     # one packed byte per pixel (VGG conv1_1): the row-per-thread kernel
    (1, 7, 7, 8, 3, 2, 1, 2),      # two bytes per pixel, stride 2, pad code 2
    (3, 6, 5, 12, 3, 1, 1, 3),     # three bytes per pixel
    (1, 8, 8, 16, 3, 1, 1, 1),     # 4-byte path
    (1, 6, 6, 64, 3, 1, 1, 0),     # 16-byte path
])
def test_im2col_bytes(B, H, W, C, k, stride, pad, pad_code):
    """dg_im2col byte layout: row (b, ho, wo), K order (r, s, c), out-of-image taps = the pad code,
    zero tail; compared with the packing of the im2col of the code tensor (numpy indexing)."""
    g = np.random.default_rng(B + H + W + C + k + pad_code)
    x = g.integers(0, 4, (B, H, W, C), dtype=np.uint8)
    Ho, Wo = (H + 2 * pad - k) // stride + 1, (W + 2 * pad - k) // stride + 1
    xpad = np.full((B, H + 2 * pad, W + 2 * pad, C), pad_code, np.uint8)
    xpad[:, pad:pad + H, pad:pad + W] = x
    cols = np.empty((B, Ho, Wo, k, k, C), np.uint8)
    for r in range(k):
        for s_ in range(k):
            cols[:, :, :, r, s_] = xpad[:, r:r + stride * Ho:stride, s_:s_ + stride * Wo:stride]
    cols = cols.reshape(B * Ho * Wo, k * k * C)
    xp, Cp = nhwc_pack(x)
    got = host(dg.im2col(xp, B, H, W, Cp, k, k, stride, pad, pad_code))
    exp = host(dg.pack_codes(torch.from_numpy(np.ascontiguousarray(cols)).to(DEV)))
    assert got.shape[0] == exp.shape[0]
    assert np.array_equal(got[:, : exp.shape[1]], exp)


@pytest.mark.parametrize("K", [1, 37, 64, 101])
def test_pack_codes4(K):
    """dg_pack_codes4: nibble k&1 of byte k>>1 (low first), zero tail, values > 15 masked and
    counted; the same bytes as the 2-bit packing of the digit sequence (c & 3, c >> 2)."""
    g = np.random.default_rng(K)
    codes = g.integers(0, 16, (9, K), dtype=np.uint8)
    codes[3, 0] = 200
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    got = host(dg.pack_codes4(torch.from_numpy(codes).to(DEV), err=err))
    assert int(err.item()) == 1
    m = codes & 15
    exp = np.zeros((9, got.shape[1]), np.uint8)
    for k in range(K):
        exp[:, k >> 1] |= (m[:, k] << (4 * (k & 1))).astype(np.uint8)
    assert np.array_equal(got, exp)
    digits = np.stack((m & 3, m >> 2), axis=2).reshape(9, 2 * K)
    assert np.array_equal(host(dg.pack_codes(torch.from_numpy(np.ascontiguousarray(digits)).to(DEV))), got)


@pytest.mark.parametrize("M,N,K", [(64, 196, 576), (130, 70, 300), (256, 384, 1152), (17, 9, 5)])
def test_gemm4_vs_oracle(M, N, K):
    """4-bit weights (16 arbitrary int8 levels) x 4-bit unsigned activations: activation-major
    Ct[n][m] equals the b-bit oracle (256-entry product table) bit for bit; the documented packing
    (digit sequence through dg_pack_codes) gives the nibble layout."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    g = np.random.default_rng(M * 7 + N + K)
    wl = _levels16(M + K)
    W = g.integers(0, 16, (M, K), dtype=np.uint8)
    A = g.integers(0, 16, (K, N), dtype=np.uint8)
    T = np.outer(wl, np.arange(16)).reshape(-1).astype(np.int32)
    w4 = dg.pack_codes4(torch.from_numpy(W).to(DEV))
    hw = host(w4)
    assert np.array_equal(hw[:, : K // 2], (W[:, 0:K - K % 2:2] | (W[:, 1:K:2] << 4)).astype(np.uint8)[:, : K // 2])
    at4 = dg.pack_codes4(torch.from_numpy(np.ascontiguousarray(A.T)).to(DEV))
    w8 = dg.expand_digits4(w4, K, wl)
    Ct = host(dg.lut_gemm4_prepared(at4, w8, N, M, K, wl))
    assert np.array_equal(Ct, oracle.lut_gemm_bits(W, A, T, 4).T)


@pytest.mark.parametrize("B,H,W,C,Cout,k,stride,pad", [(2, 9, 7, 32, 64, 3, 1, 1), (1, 12, 12, 64, 32, 3, 2, 1),
                                                       (2, 6, 6, 32, 16, 1, 1, 0), (1, 8, 8, 8, 8, 3, 1, 1)])
def test_conv4_vs_oracle(B, H, W, C, Cout, k, stride, pad):
    """4-bit NHWC conv (implicit GEMM over 2C digit channels where C/2 bytes is a power of two >= 16,
    direct 1x1, im2col otherwise) vs the b-bit direct-conv oracle; int32 and fused requant."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    g = np.random.default_rng(B + H + C + Cout + k)
    wl = _levels16(C + Cout)
    x = g.integers(0, 16, (B, H, W, C), dtype=np.uint8)
    wc = g.integers(0, 16, (Cout, k, k, C), dtype=np.uint8)
    T = np.outer(wl, np.arange(16)).reshape(-1).astype(np.int32)
    exp = oracle.conv2d_direct_bits(x, wc, T, stride, pad, 4).reshape(-1, Cout)
    # NHWC activations are contiguous C/2 bytes per pixel: pack the whole tensor as one row
    nb = B * H * W * C // 2
    x4 = dg.pack_codes4(torch.from_numpy(x.reshape(1, -1)).to(DEV))[0, :nb].reshape(B * H * W, C // 2).contiguous()
    w4 = dg.pack_codes4(torch.from_numpy(wc.reshape(Cout, -1)).to(DEV))
    w8 = dg.expand_digits4(w4, k * k * C, wl)
    p = dg.conv_params(B, H, W, C, Cout, k, k, stride, pad, 0, ldw=w4.shape[1])
    ws = torch.zeros(max(1, dg.conv_workspace_size(dg.conv_params(B, H, W, 2 * C, Cout, k, k, stride, pad, 0))),
                     dtype=torch.uint8, device=DEV)
    got = host(dg.lut_conv2d4_prepared(x4, w8, wl, p, ws=ws))
    assert np.array_equal(got, exp)
    rq = dg.Requant(3000, 20, 0, 0, 3, bias=torch.full((Cout,), int(-exp.mean()), dtype=torch.int32, device=DEV))
    codes = dg.lut_conv2d4_prepared(x4, w8, wl, p, rq=rq, ws=ws)
    gotc = oracle.unpack_codes(host(codes), exp.shape[0], Cout, codes.shape[1])
    bias = np.full(Cout, int(-exp.mean()), np.int32)
    assert np.array_equal(gotc, oracle.requantize(exp, 3000, 20, 0, 0, 3, bias=bias, bias_axis=0))


def test_digits4_rejects():
    if not _tc_available():
        pytest.skip("tc unavailable")
    w4 = dg.pack_codes4(torch.zeros((4, 64), dtype=torch.uint8, device=DEV))
    with pytest.raises(dg.DGError, match="RANGE"):
        dg.expand_digits4(w4, 64, [40] + [0] * 15)      # 4 x 40 > 127


def test_conv_window_default_with_residual_and_bias():
    """A 3x3 C = 64 conv large enough (>= 2 waves of padded-pixel tiles) to take the shifted-window
    kernel by default (tile + pair mode) with an identity residual over packed codes and a
    per-channel bias: the window path's general epilogue equals O-RES / O-REQ."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    lut = dg.build_lut(WL, AL, 8)
    T = oracle.build_lut16(WL, AL)
    g = np.random.default_rng(88)
    B, H, C = 12, 56, 64
    x = g.integers(0, 4, (B, H, H, C), dtype=np.uint8)
    w = g.integers(0, 4, (C, 3, 3, C), dtype=np.uint8)
    xp, Cp = nhwc_pack(x)
    wp = conv_weights_pack(w, Cp)
    w8 = dg.expand_operand(wp, 9 * Cp, WL)
    p = dg.conv_params(B, H, H, C, C, 3, 3, 1, 1, 0, ldw=wp.shape[1])
    ws = torch.empty(dg.conv_workspace_size(p), dtype=torch.uint8, device=DEV)
    acc = oracle.conv2d_direct(x, w, T, 1, 1, 0).reshape(-1, C)
    assert np.array_equal(host(dg.lut_conv2d_prepared(xp, w8, lut, p, ws=ws)), acc)
    bias = g.integers(-300, 300, C).astype(np.int32)
    rq = dg.Requant(mult=15000, shift=20, zp=0, res_codes=xp, res_mult=29, res_levels=AL,
                    bias=torch.from_numpy(bias).to(DEV), bias_axis=0)
    out = dg.lut_conv2d_prepared(xp, w8, lut, p, rq=rq, ws=ws)
    r = (np.array(AL)[x.reshape(-1, C)] * 29).astype(np.int32)
    exp = oracle.requantize(acc, 15000, 20, 0, 0, 3, res=r, bias=bias, bias_axis=0)
    assert np.array_equal(oracle_codes_of(out, exp.shape[0], C), exp)


# ---- every TS-kernel instance of the auto dispatch (and the forced ablation forms), tag-checked ----
INSTANCES = [  # np (pixels), nq (channels), K, options, tags the instance must carry
    (300, 64, 64, {}, ["bn=64 epi=8 unp=8 kst=128"]),
    (300, 64, 256, {}, ["bn=64 epi=8 unp=8 kst=256"]),
    (300, 128, 128, {}, ["bn=128 epi=8 unp=4 kst=128"]),
    (300, 128, 256, {}, ["bn=128 epi=8 unp=4 kst=256"]),
    (300, 256, 64, {}, ["bn=256 epi=8 unp=4 kst=128 asm", "offs=1"]),
    (260, 512, 256, {}, ["bn=256 epi=8 unp=4 kst=128 asm", "offs=1"]),
    (300, 256, 64, {"offs": 0}, ["bn=256 epi=8 unp=4 kst=128 asm", "offs=0"]),
    (300, 768, 64, {}, ["asm", "offs=0"]),                               # 3 column tiles: table path
    (300, 256, 3200, {}, ["bn=256 epi=4 unp=8 kst=128", "sk=1"]),
    (300, 128, 1152, {}, ["bn=128 epi=4 unp=8 kst=256"]),
    (300, 64, 1152, {}, ["bn=64 epi=4 unp=8 kst=256"]),
    (300, 96, 1152, {"kst": 128}, ["bn=128 epi=4 unp=8 kst=128"]),
    (300, 64, 1000, {"kst": 128}, ["bn=64 epi=4 unp=8 kst=128"]),
    (300, 100, 256, {"bn64_short": 1}, ["bn=64 epi=8 unp=8 kst=256"]),
    (300, 256, 3200, {"bn256": 0}, ["bn=128 epi=4 unp=8 kst=256"]),
    (300, 256, 64, {"asm": 0}, ["bn=128 epi=8 unp=4 kst=128"]),
    (300, 128, 1152, {"f16": 0}, ["f16=0"]),
    (300, 128, 1152, {"bres": 0}, ["bres=0"]),
    (300, 128, 576, {"pdl": 0, "early_weights": 1}, ["early=1"]),
    # B multicast across 2-CTA clusters (even row-block count and raster group, streamed B)
    (512, 1280, 1024, {"bmc": 1}, ["epi=4 unp=8", "bmc=1"]),
    (1000, 2048, 2048, {"bmc": 1}, ["epi=4 unp=8", "bmc=1"]),         # ragged last row block
    (512, 1280, 1024, {}, ["epi=4 unp=8", "bmc=0"]),
    (300, 1280, 1024, {"bmc": 1}, ["bmc=0"]),                           # odd row-block count
]


@pytest.mark.parametrize("big", [False, True])
def test_asm_offset_mma_and_fallback(big):
    """Short-K shared-memory-A instance with the per-column requant offsets written into the
    accumulator by one MMA per tile (n = 127 q + r): bit-exact against the oracle; with offsets
    beyond that range (|n| > 16192, still within the 16-bit form) every CTA falls back to the
    offset-table path, also bit-exact."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    np_, nq, K = 700, 512, 64
    g = np.random.default_rng(5 + big)
    A = g.integers(0, 4, (np_, K), dtype=np.uint8)
    Wt = g.integers(0, 4, (nq, K), dtype=np.uint8)
    acc = oracle.lut_gemm(Wt, np.ascontiguousarray(A.T), oracle.build_lut16(WL, AL)).T
    a_p, w8 = gpu_pack(A), dg.expand_operand(gpu_pack(Wt, weights=True), K, WL)
    lut_t = dg.build_lut(AL, WL, 8)
    base = 20000 if big else -int(np.round(acc.mean()))
    bias = (base + g.integers(-300, 300, nq)).astype(np.int32)
    mult = 40000
    rq = dg.Requant(mult, 20, 1, 0, 3, bias=torch.from_numpy(bias).to(DEV), bias_axis=0)
    dg.reset_options()
    codes = dg.lut_gemm_prepared(a_p, w8, np_, nq, K, lut_t, rq=rq)
    assert "asm" in dg.last_kernel() and "offs=1" in dg.last_kernel(), dg.last_kernel()
    exp = oracle.requantize(np.ascontiguousarray(acc), mult, 20, 1, 0, 3, bias=bias, bias_axis=0)
    assert np.array_equal(oracle_codes_of(codes, np_, nq), exp)
    if not big:
        assert len(np.unique(exp)) == 4   # (every code occurs: a real test of the thresholds)


@pytest.mark.parametrize("np_,nq,K,opts,tags", INSTANCES)
def test_dispatch_instances_vs_oracle(np_, nq, K, opts, tags):
    """Each TS-kernel instance (template / runtime mode named by dg_last_kernel), int32 and fused
    requant (per-column bias) in the conv orientation, bit-exact against the oracle; ragged rows."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    g = np.random.default_rng(np_ + 7 * nq + K)
    A = g.integers(0, 4, (np_, K), dtype=np.uint8)      # activations (pixels), K-major
    Wt = g.integers(0, 4, (nq, K), dtype=np.uint8)      # weights [channel][K]
    acc = oracle.lut_gemm(Wt, np.ascontiguousarray(A.T), oracle.build_lut16(WL, AL)).T
    a_p, w8 = gpu_pack(A), dg.expand_operand(gpu_pack(Wt, weights=True), K, WL)
    lut_t = dg.build_lut(AL, WL, 8)
    bias = (-int(np.round(acc.mean())) + g.integers(-30, 30, nq)).astype(np.int32)
    rq = dg.Requant(20000 if K < 1024 else 9000, 20, 1, 0, 3, bias=torch.from_numpy(bias).to(DEV), bias_axis=0)
    dg.reset_options()
    with dg.options(**opts):
        C = dg.lut_gemm_prepared(a_p, w8, np_, nq, K, lut_t)
        tag = dg.last_kernel()
        codes = dg.lut_gemm_prepared(a_p, w8, np_, nq, K, lut_t, rq=rq)
        tag_rq = dg.last_kernel()
        assert tag_rq.split(" f16=")[0] == tag.split(" f16=")[0]
        tag = tag_rq
    for t in tags:
        assert t in tag, (t, tag)
    assert np.array_equal(host(C), acc)
    exp = oracle.requantize(np.ascontiguousarray(acc), rq.mult, 20, 1, 0, 3, bias=bias, bias_axis=0)
    assert np.array_equal(oracle_codes_of(codes, np_, nq), exp)


# ---- convolution on the block-scaled FP4 path (dg_lut_conv2d_f4_prepared) ----
F4_CONVS = [  # B, H, W, C, Cout, k, stride, pad, pad_code
    (2, 9, 9, 64, 128, 1, 1, 0, 0),      # direct 1x1 (TMA slots of the NHWC tensor), 64 channels
    (3, 7, 7, 256, 256, 1, 1, 0, 0),     # direct, 2 column tiles
    (1, 6, 5, 512, 200, 1, 1, 0, 0),     # direct, ragged Cout and rows
    (2, 10, 10, 64, 128, 3, 1, 1, 0),    # implicit 3x3 gather, 4 taps per stage
    (2, 9, 11, 128, 128, 3, 2, 1, 2),    # implicit stride 2, pad code 2
    (1, 8, 8, 256, 384, 3, 1, 1, 1),     # implicit, 1 tap per stage, 3 column tiles, pad code 1
    (2, 12, 12, 256, 128, 1, 2, 0, 0),   # implicit 1x1 stride 2 (downsample)
    (1, 7, 7, 512, 136, 3, 1, 1, 3),     # ragged Cout, K = 4608
    (2, 9, 9, 256, 64, 1, 1, 0, 0),      # direct into 64 channels (one 64-wide tile)
    (2, 10, 10, 64, 64, 3, 1, 1, 2),     # implicit 3x3 64 -> 64, K = 576
]


# (tile width, epilogue arrangement): 64-wide tiles run 8 epilogue warps only, two CTAs per SM
# ("ct2") 128-wide tiles only
F4_BN_EPI = [(64, 8), (128, 4), (128, 8), (128, "ct2"), (256, 4), (256, 8)]


@pytest.mark.parametrize("omma", [0, 1])
@pytest.mark.parametrize("bn,epi", F4_BN_EPI)
@pytest.mark.parametrize("wl", [(-2, -1, 0, 1), (-12, -3, 4, 8)])
@pytest.mark.parametrize("B,H,W,C,Cout,k,stride,pad,pad_code", F4_CONVS)
def test_conv_f4_vs_oracle(wl, B, H, W, C, Cout, k, stride, pad, pad_code, bn, epi, omma):
    """FP4 conv kernel vs O-CONV on the three tile widths (64 channels, four accumulators; 128, two;
    256, one) and
    both epilogue arrangements (4 warps; 8 warps splitting the 256-wide tiles' columns or owning
    alternate 128-wide tiles): int32 output, fused 16-bit requant with a per-channel bias, a
    uniform-offset requant without bias, and a bias whose 16-bit offsets overflow (exact path)."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    wl = list(wl)
    lut = dg.build_lut(wl, AL, 8)
    T = oracle.build_lut16(wl, AL)
    g = np.random.default_rng(B + H + W + C + Cout + k + pad_code + wl[0])
    x = g.integers(0, 4, (B, H, W, C), dtype=np.uint8)
    w = g.integers(0, 4, (Cout, k, k, C), dtype=np.uint8)
    exp = oracle.conv2d_direct(x, w, T, stride, pad, pad_code).reshape(-1, Cout)
    xp, Cp = nhwc_pack(x)
    wp = conv_weights_pack(w, Cp)
    w4 = dg.expand_operand_f4(wp, k * k * Cp, wl)
    p = dg.conv_params(B, H, W, Cp, Cout, k, k, stride, pad, pad_code, ldw=wp.shape[1])
    dg.reset_options()
    ct = 2 if epi == "ct2" else 1
    epi = 4 if epi == "ct2" else epi
    # (f4_win=0: the gathered / direct instances; the shifted-window ones, the default for the 3x3
    # s1 convs over 64 / 128 channels with resident weights, are test_conv_f4_window_vs_oracle's)
    with dg.options(f4_bn=bn, f4_epi=epi, f4_omma=omma, f4_ct=ct, f4_win=0):
        _conv_f4_cases(xp, w4, lut, p, exp, Cout, g, bn, epi)
        assert (" ct=2 " in dg.last_kernel()) == (ct == 2), dg.last_kernel()
        assert dg.last_kernel().endswith(f" omma={omma}"), dg.last_kernel()


F4_STRIDED_1X1 = [  # B, H, W, C, Cout, stride, pad_code: strided 1x1 convs (downsample)
    (2, 12, 12, 256, 128, 2, 0),
    (1, 13, 11, 128, 256, 2, 1),     # odd input: Ho = 7, Wo = 6 (the traversal skips the last column)
    (3, 14, 14, 512, 64, 2, 0),
    (2, 10, 10, 64, 128, 3, 0),      # stride 3, 16-byte pixels (half of every 128-byte slot row is beyond C)
    (4, 28, 28, 1024, 256, 2, 0),    # K = 1024: two packed slots per tile, tiles across images
]


@pytest.mark.parametrize("i2c", [0, 1])
@pytest.mark.parametrize("B,H,W,C,Cout,stride,pad_code", F4_STRIDED_1X1)
def test_conv_f4_strided_1x1_vs_oracle(B, H, W, C, Cout, stride, pad_code, i2c):
    """Strided 1x1 convs on the FP4 kernel: the direct path whose slots arrive through an
    im2col-mode TMA tensor map (element strides = the conv stride; option f4_i2c) and the per-thread
    gather, vs O-CONV (int32 and fused requant), the instance asserted by its tag."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    wl = [-2, -1, 0, 1]
    lut = dg.build_lut(wl, AL, 8)
    T = oracle.build_lut16(wl, AL)
    g = np.random.default_rng(B + H + W + C + Cout + stride)
    x = g.integers(0, 4, (B, H, W, C), dtype=np.uint8)
    w = g.integers(0, 4, (Cout, 1, 1, C), dtype=np.uint8)
    exp = oracle.conv2d_direct(x, w, T, stride, 0, pad_code).reshape(-1, Cout)
    xp, Cp = nhwc_pack(x)
    wp = conv_weights_pack(w, Cp)
    w4 = dg.expand_operand_f4(wp, Cp, wl)
    p = dg.conv_params(B, H, W, Cp, Cout, 1, 1, stride, 0, pad_code, ldw=wp.shape[1])
    dg.reset_options()
    with dg.options(f4_i2c=i2c):
        out = dg.lut_conv2d_f4_prepared(xp, w4, lut, p)
        tag = dg.last_kernel()
        assert (" direct=1 i2c " in tag) == (i2c == 1) and (" direct=0 " in tag) == (i2c == 0), tag
        assert np.array_equal(host(out), exp)
        bias = (-int(np.round(exp.mean())) + g.integers(-40, 40, Cout)).astype(np.int32)
        mult = max(1, int(round((1 << 20) * 1.2 / max(1.0, float(exp.std())))))
        rq = dg.Requant(mult, 20, 1, 0, 3, bias=torch.from_numpy(bias).to(DEV), bias_axis=0)
        codes = dg.lut_conv2d_f4_prepared(xp, w4, lut, p, rq=rq)
        expc = oracle.requantize(exp, mult, 20, 1, 0, 3, bias=bias, bias_axis=0)
        assert np.array_equal(oracle_codes_of(codes, exp.shape[0], Cout), expc)


F4_1X1_WIN = [  # B, H, W, C, Cout: 1x1 stride-1 convs into 64 / 128 channels (K <= 256)
    (2, 10, 10, 64, 64),
    (1, 9, 7, 128, 128),       # 63 rows: one ragged pair
    (3, 14, 14, 256, 64),      # 588 rows: pairs across images, ragged last pair
    (2, 28, 28, 256, 128),     # many pairs per CTA: window ring reuse
    (1, 5, 5, 64, 100),        # ragged Cout (exact epilogue path on the last columns)
]


@pytest.mark.parametrize("B,H,W,C,Cout", F4_1X1_WIN)
def test_conv_f4_1x1_window_pairs_vs_oracle(B, H, W, C, Cout):
    """1x1 stride-1 convs on the FP4 kernel's window-pair form (option f4_w1x1 = 2: a pair's 256 pixel
    rows are the shared-memory A window, resident weights, two 128-row accumulators per hand-off)
    vs O-CONV: int32 and the fused requant, the instance asserted by its tag."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    wl = [-2, -1, 0, 1]
    lut = dg.build_lut(wl, AL, 8)
    T = oracle.build_lut16(wl, AL)
    g = np.random.default_rng(B + H + W + C + Cout)
    x = g.integers(0, 4, (B, H, W, C), dtype=np.uint8)
    w = g.integers(0, 4, (Cout, 1, 1, C), dtype=np.uint8)
    exp = oracle.conv2d_direct(x, w, T, 1, 0, 0).reshape(-1, Cout)
    xp, Cp = nhwc_pack(x)
    wp = conv_weights_pack(w, Cp)
    w4 = dg.expand_operand_f4(wp, Cp, wl)
    p = dg.conv_params(B, H, W, Cp, Cout, 1, 1, 1, 0, 0, ldw=wp.shape[1])
    dg.reset_options()
    with dg.options(f4_w1x1=2):   # (2: every channel count; the default takes C = 64 only)
        out = dg.lut_conv2d_f4_prepared(xp, w4, lut, p)
        assert " win1x1 " in dg.last_kernel(), dg.last_kernel()
        assert np.array_equal(host(out), exp)
        if Cout % 4 == 0:
            bias = (-int(np.round(exp.mean())) + g.integers(-40, 40, Cout)).astype(np.int32)
            mult = max(1, int(round((1 << 20) * 1.2 / max(1.0, float(exp.std())))))
            rq = dg.Requant(mult, 20, 1, 0, 3, bias=torch.from_numpy(bias).to(DEV), bias_axis=0)
            codes = dg.lut_conv2d_f4_prepared(xp, w4, lut, p, rq=rq)
            assert " win1x1 " in dg.last_kernel(), dg.last_kernel()
            expc = oracle.requantize(exp, mult, 20, 1, 0, 3, bias=bias, bias_axis=0)
            assert np.array_equal(oracle_codes_of(codes, exp.shape[0], Cout), expc)


def _conv_f4_cases(xp, w4, lut, p, exp, Cout, g, bn, epi):
    out = dg.lut_conv2d_f4_prepared(xp, w4, lut, p)
    assert dg.last_kernel().startswith(f"f4conv bn={bn} ") and f" epi={epi} " in dg.last_kernel(), dg.last_kernel()
    assert np.array_equal(host(out), exp)
    if Cout % 4:
        return
    mu = int(np.round(exp.mean()))
    bias = (-mu + g.integers(-40, 40, Cout)).astype(np.int32)
    mult = max(1, int(round((1 << 20) * 1.2 / max(1.0, float(exp.std())))))
    for b in (bias, None, np.full(Cout, 30000, np.int32)):
        rq = dg.Requant(mult, 20, 1, 0, 3, bias=None if b is None else torch.from_numpy(b).to(DEV), bias_axis=0)
        try:
            codes = dg.lut_conv2d_f4_prepared(xp, w4, lut, p, rq=rq)
        except dg.DGError as e:   # (no 16-bit form of these parameters: the caller takes the int8 path)
            assert "UNSUPPORTED" in str(e)
            continue
        expc = oracle.requantize(exp, mult, 20, 1, 0, 3, bias=b, bias_axis=0)
        assert np.array_equal(oracle_codes_of(codes, exp.shape[0], Cout), expc)


F4_WIN_CONVS = [  # B, H, W, C, Cout, pad_code (3x3 / stride 1 / pad 1)
    (2, 10, 10, 64, 64, 0),
    (3, 7, 9, 128, 256, 1),
    (1, 20, 30, 64, 200, 2),      # ragged Cout
    (2, 5, 5, 128, 128, 3),       # tiles mostly padding
    (4, 28, 28, 64, 128, 0),      # many tiles per CTA: window ring reuse
    (1, 56, 56, 128, 256, 1),
    (1, 3, 200, 64, 64, 2),       # wide rows: 3 window rows per fill thread
]


@pytest.mark.parametrize("wbres", [0, 1])   # (1: pair mode too where the tiles are 64 / 128 wide)
@pytest.mark.parametrize("omma", [0, 1])
@pytest.mark.parametrize("wl", [(-2, -1, 0, 1), (-12, -3, 4, 8)])
@pytest.mark.parametrize("B,H,W,C,Cout,pad_code", F4_WIN_CONVS)
def test_conv_f4_window_vs_oracle(B, H, W, C, Cout, pad_code, omma, wl, wbres):
    """FP4 conv, shifted-window mode (each padded input pixel unpacked once per tile into a shared-
    memory window; the 9 taps are row-shifted views, shared-memory MMAs) vs O-CONV: int32 and the
    fused requant with a per-channel bias (levels -2..1: every case has a 16-bit requant form), the
    instance asserted by its tag; with and without resident weights (option f4_wbres: one column
    block whose weight stages fit the B ring is loaded once, one MMA hand-off per tile)."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    wl = list(wl)
    lut = dg.build_lut(wl, AL, 8)
    T = oracle.build_lut16(wl, AL)
    g = np.random.default_rng(B + H + W + C + Cout + pad_code)
    x = g.integers(0, 4, (B, H, W, C), dtype=np.uint8)
    w = g.integers(0, 4, (Cout, 3, 3, C), dtype=np.uint8)
    exp = oracle.conv2d_direct(x, w, T, 1, 1, pad_code).reshape(-1, Cout)
    xp, Cp = nhwc_pack(x)
    wp = conv_weights_pack(w, Cp)
    w4 = dg.expand_operand_f4(wp, 9 * Cp, wl)
    p = dg.conv_params(B, H, W, Cp, Cout, 3, 3, 1, 1, pad_code, ldw=wp.shape[1])
    dg.reset_options()
    bnt = 256 if Cout % 256 == 0 else (64 if Cout <= 64 else 128)
    resident = wbres == 1 and -(-Cout // bnt) == 1 and -(-9 * Cp // 256) <= (3 if bnt == 256 else 6)
    with dg.options(f4_win=1, f4_omma=omma, f4_wbres=wbres):
        out = dg.lut_conv2d_f4_prepared(xp, w4, lut, p)
        tag = dg.last_kernel()
        assert " win " in tag, tag
        assert ("wbres" in tag) == resident, tag
        assert ("wpair" in tag) == (resident and bnt <= 128), tag
        assert np.array_equal(host(out), exp)
        if Cout % 4 == 0:
            bias = (-int(np.round(exp.mean())) + g.integers(-40, 40, Cout)).astype(np.int32)
            mult = max(1, int(round((1 << 20) * 1.2 / max(1.0, float(exp.std())))))
            rq = dg.Requant(mult, 20, 1, 0, 3, bias=torch.from_numpy(bias).to(DEV), bias_axis=0)
            try:
                codes = dg.lut_conv2d_f4_prepared(xp, w4, lut, p, rq=rq)
            except dg.DGError as e:   # (no 16-bit form of these parameters: the caller takes the int8 path)
                assert "UNSUPPORTED" in str(e) and wl[0] == -12
                return
            assert " win " in dg.last_kernel(), dg.last_kernel()
            expc = oracle.requantize(exp, mult, 20, 1, 0, 3, bias=bias, bias_axis=0)
            assert np.array_equal(oracle_codes_of(codes, exp.shape[0], Cout), expc)


def test_conv_f4_accumulator_origin_at_the_bound():
    """The FP4 conv accumulates from 1.5 * 2^23: at the largest K the API admits (K * 36 < 2^22 for
    weight level -12 and activation level 3), all-max products first then a random tail, positive and
    negative sums must stay exact; one code more is refused."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    wl = [-12, -3, 4, 8]
    lut = dg.build_lut(wl, AL, 8)
    T = oracle.build_lut16(wl, AL)
    K = ((1 << 22) - 1) // 36 // 64 * 64          # 1x1 conv over K channels
    B, H, W, Cout = 1, 1, 5, 128
    g = np.random.default_rng(9)
    x = g.integers(0, 4, (B, H, W, K), dtype=np.uint8)
    x[0, 0, :3, : K - 64] = 3
    w = g.integers(0, 4, (Cout, 1, 1, K), dtype=np.uint8)
    w[::2, 0, 0, : K - 64] = 0                    # level -12 (negative extreme)
    w[1::4, 0, 0, : K - 64] = 3                   # level 8
    exp = oracle.conv2d_direct(x, w, T, 1, 0, 0).reshape(-1, Cout)
    assert exp.min() < -(1 << 21) and exp.max() > (1 << 20)
    xp, _ = nhwc_pack(x)
    wp = conv_weights_pack(w, K)
    w4 = dg.expand_operand_f4(wp, K, wl)
    p = dg.conv_params(B, H, W, K, Cout, 1, 1, 1, 0, 0, ldw=wp.shape[1])
    assert np.array_equal(host(dg.lut_conv2d_f4_prepared(xp, w4, lut, p)), exp)
    K2 = K + 64 * 60
    p2 = dg.conv_params(1, 1, 1, K2, 8, 1, 1, 1, 0, 0)
    w2 = dg.expand_operand_f4(gpu_pack(np.zeros((8, K2), np.uint8), weights=True), K2, wl)
    with pytest.raises(dg.DGError, match="OVERFLOW"):
        dg.lut_conv2d_f4_prepared(gpu_pack(np.zeros((1, K2), np.uint8))[:, : K2 // 4].contiguous(), w2, lut, p2)


# ---- float-valued tables (dg_lut_gemm_f32, fixed-point digits on the one-hot tensor-core form) ----
F32_Q = 127 * (65536 + 256 + 1)


@pytest.mark.parametrize("kind", ["random", "product", "dyadic", "tiny"])
@pytest.mark.parametrize("M,N,K", [(64, 196, 576), (130, 70, 1000), (7, 300, 33)])
def test_gemm_float_table_vs_fp64_oracle(kind, M, N, K):
    """fp32 result within the stated bound of the fp64 oracle (Q24):
    |C - C64| <= K max|T| / Q + 2^-24 |C64|; exact (up to the fp32 rounding) for dyadic entries."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    g = np.random.default_rng(M + N + K + len(kind))
    if kind == "random":
        T = g.normal(size=16) * 10.0 ** g.integers(-2, 3, 16)
    elif kind == "product":    # non-uniform quantiser levels: T = wl (x) al
        wl, al = np.sort(g.normal(size=4)), np.sort(np.abs(g.normal(size=4)))
        T = np.outer(wl, al).reshape(-1)
    elif kind == "dyadic":     # multiples of 2^-6 below 2^13: exactly representable in the fixed point
        T = g.integers(-2 ** 19, 2 ** 19, 16) / 64.0
    else:
        T = g.normal(size=16) * 1e-30
    T32 = T.astype(np.float32).astype(np.float64)
    W = g.integers(0, 4, (M, K), dtype=np.uint8)
    A = g.integers(0, 4, (K, N), dtype=np.uint8)
    C = host(dg.lut_gemm_f32(gpu_pack(W, weights=True), gpu_pack(np.ascontiguousarray(A.T)), M, N, K, T32)).astype(np.float64)
    assert dg.last_kernel().startswith("f32 table")
    C64 = oracle.lut_gemm_f64(W, A, T32)
    tol = K * np.abs(T32).max() / F32_Q + 2.0 ** -24 * np.abs(C64)
    if kind == "dyadic":
        tol = 2.0 ** -24 * np.abs(C64)
    assert np.all(np.abs(C - C64) <= tol), np.max(np.abs(C - C64) - tol)


@pytest.mark.parametrize("M,N,K", [(64, 196, 576), (33, 70, 301)])
def test_gemm3_bit_codes_in_4bit_storage(M, N, K):
    """3-bit operands (Table 2: a 6-bit index into a 64-entry table) on the 4-bit path:
    3-bit codes are 4-bit codes 0..7 (levels 8..15 unused); product table wl (x) {0..7}, vs the
    b-bit oracle with bits = 3."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    g = np.random.default_rng(M + N + K + 3)
    wl8 = g.integers(-31, 32, 8).astype(np.int32)
    wl16 = np.concatenate([wl8, np.zeros(8, np.int32)])
    W = g.integers(0, 8, (M, K), dtype=np.uint8)
    A = g.integers(0, 8, (K, N), dtype=np.uint8)
    T3 = np.outer(wl8, np.arange(8)).reshape(-1).astype(np.int32)   # index (w << 3) | a
    w4 = dg.pack_codes4(torch.from_numpy(W).to(DEV))
    at4 = dg.pack_codes4(torch.from_numpy(np.ascontiguousarray(A.T)).to(DEV))
    Ct = host(dg.lut_gemm4_prepared(at4, dg.expand_digits4(w4, K, wl16), N, M, K, wl16))
    assert np.array_equal(Ct, oracle.lut_gemm_bits(W, A, T3, 3).T)


@pytest.mark.parametrize("kind", ["random", "nonaffine_product", "three_bit"])
@pytest.mark.parametrize("M,N,K", [(64, 196, 576), (33, 70, 301)])
def test_gemm4_general_table_onehot(kind, M, N, K):
    """Any 256-entry int8 table over 4-bit codes (Table 2) on the one-hot K' = 16K path, vs the
    b-bit oracle: random non-product tables, products with NON-affine activation levels (which the
    digit path cannot take) and 3-bit tables embedded in 4-bit codes; int32 and fused requant."""
    if not _tc_available():
        pytest.skip("tc unavailable")
    g = np.random.default_rng(M + N + K + len(kind))
    if kind == "random":
        T = g.integers(-127, 128, 256).astype(np.int32)
        W = g.integers(0, 16, (M, K), dtype=np.uint8)
        A = g.integers(0, 16, (K, N), dtype=np.uint8)
        exp = oracle.lut_gemm_bits(W, A, T, 4)
    elif kind == "nonaffine_product":
        wl = g.integers(-11, 12, 16)
        al = np.sort(g.integers(0, 12, 16))                  # non-uniform activation levels
        T = np.outer(wl, al).reshape(-1).astype(np.int32)
        W = g.integers(0, 16, (M, K), dtype=np.uint8)
        A = g.integers(0, 16, (K, N), dtype=np.uint8)
        exp = oracle.lut_gemm_bits(W, A, T, 4)
    else:
        T3 = g.integers(-127, 128, 64).astype(np.int32)    # 3-bit: 6-bit index (w << 3) | a
        T = np.zeros(256, np.int32)
        for w in range(8):
            for a in range(8):
                T[(w << 4) | a] = T3[(w << 3) | a]
        W = g.integers(0, 8, (M, K), dtype=np.uint8)
        A = g.integers(0, 8, (K, N), dtype=np.uint8)
        exp = oracle.lut_gemm_bits(W, A, T3, 3)
    w4 = dg.pack_codes4(torch.from_numpy(W).to(DEV))
    at4 = dg.pack_codes4(torch.from_numpy(np.ascontiguousarray(A.T)).to(DEV))
    C = host(dg.lut_gemm4_table(w4, at4, M, N, K, T))
    assert np.array_equal(C, exp)
    mu = int(np.round(exp.mean()))
    rq = dg.Requant(max(1, int((1 << 20) / max(1.0, exp.std()))), 20, 1, 0, 3,
                    bias=torch.full((N,), -mu, dtype=torch.int32, device=DEV), bias_axis=0)
    codes = dg.lut_gemm4_table(w4, at4, M, N, K, T, rq=rq)
    expc = oracle.requantize(exp, rq.mult, 20, 1, 0, 3, bias=np.full(N, -mu, np.int32), bias_axis=0)
    assert np.array_equal(oracle_codes_of(codes, M, N), expc)
