"""Small cases covering every kernel instance, for compute-sanitizer (memcheck / racecheck / synccheck).

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py [filter]

Each case forces one instance through dg_set_option, runs it once, checks the result against the
oracle (so the sanitizer's perturbed scheduling is also a parity run) and prints the instance tag.
Shapes are small (a few tiles, ragged) because the sanitizer serialises and instruments every
access."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2304_09049_b200 import dg  # noqa: E402

WL, AL = [-2, -1, 0, 1], [0, 1, 2, 3]
DEV = "cuda"


def pack(codes, weights=False):
    return dg.pack_codes(torch.from_numpy(np.ascontiguousarray(codes, dtype=np.uint8)).to(DEV), weights=weights)


def codes_of(t, rows, cols):
    h = t.cpu().numpy()
    return oracle.unpack_codes(h, rows, cols, h.shape[1])


def gemm_case(np_, nq, K, opts, seed=1):
    g = np.random.default_rng(seed + np_ + nq + K)
    A = g.integers(0, 4, (np_, K), dtype=np.uint8)
    Wt = g.integers(0, 4, (nq, K), dtype=np.uint8)
    acc = oracle.lut_gemm(Wt, np.ascontiguousarray(A.T), oracle.build_lut16(WL, AL)).T
    a_p, w8 = pack(A), dg.expand_operand(pack(Wt, True), K, WL)
    lut_t = dg.build_lut(AL, WL, 8)
    bias = (-int(np.round(acc.mean())) + g.integers(-30, 30, nq)).astype(np.int32)
    rq = dg.Requant(20000, 20, 1, 0, 3, bias=torch.from_numpy(bias).to(DEV), bias_axis=0)
    with dg.options(**opts):
        C = dg.lut_gemm_prepared(a_p, w8, np_, nq, K, lut_t)
        tag = dg.last_kernel()
        codes = dg.lut_gemm_prepared(a_p, w8, np_, nq, K, lut_t, rq=rq)
    torch.cuda.synchronize()
    ok = np.array_equal(C.cpu().numpy(), acc) and np.array_equal(
        codes_of(codes, np_, nq), oracle.requantize(np.ascontiguousarray(acc), 20000, 20, 1, 0, 3, bias=bias))
    return tag, ok


def conv_case(B, H, W, C, Cout, k, stride, opts, res=False, ws_fill=None, seed=2):
    g = np.random.default_rng(seed + B + H + C + Cout + k)
    x = g.integers(0, 4, (B, H, W, C), dtype=np.uint8)
    w = g.integers(0, 4, (Cout, k, k, C), dtype=np.uint8)
    pad = k // 2
    T = oracle.build_lut16(WL, AL)
    exp = oracle.conv2d_direct(x, w, T, stride, pad, 0).reshape(-1, Cout)
    xp = pack(x.reshape(-1, C))[:, : C // 4].contiguous()
    wp = pack(w.reshape(Cout, -1), True)
    w8 = dg.expand_operand(wp, k * k * C, WL)
    p = dg.conv_params(B, H, W, C, Cout, k, k, stride, pad, 0, ldw=wp.shape[1])
    ws = torch.full((dg.conv_workspace_size(p),), ws_fill if ws_fill is not None else 0, dtype=torch.uint8, device=DEV)
    lut = dg.build_lut(WL, AL, 8)
    rqkw = {}
    r = None
    if res:
        r = (np.array(AL)[x.reshape(-1, C)] * 29).astype(np.int32)
        rqkw = dict(res_codes=xp, res_mult=29, res_levels=AL)
    with dg.options(**opts):
        out = dg.lut_conv2d_prepared(xp, w8, lut, p, ws=ws)
        tag = dg.last_kernel()
        codes = dg.lut_conv2d_prepared(xp, w8, lut, p, ws=ws, rq=dg.Requant(15000, 20, 0, **rqkw))
    torch.cuda.synchronize()
    ok = np.array_equal(out.cpu().numpy(), exp) and np.array_equal(
        codes_of(codes, exp.shape[0], Cout), oracle.requantize(exp, 15000, 20, 0, 0, 3, res=r))
    return tag, ok


def f4_case():
    g = np.random.default_rng(3)
    M, N, K = 250, 140, 600
    W = g.integers(0, 4, (M, K), dtype=np.uint8)
    A = g.integers(0, 4, (K, N), dtype=np.uint8)
    lut = dg.build_lut(WL, AL, 8)
    C = dg.lut_gemm_f4(dg.expand_operand_f4(pack(W, True), K, WL), pack(A.T), M, N, K, lut)
    torch.cuda.synchronize()
    return dg.last_kernel(), np.array_equal(C.cpu().numpy(), oracle.lut_gemm(W, A, oracle.build_lut16(WL, AL)))


def f4conv_case(B, H, W, C, Cout, k, stride, opts, seed=6):
    """FP4 conv kernel instance (dg_lut_conv2d_f4_prepared): int32 and the fused 16-bit requant."""
    g = np.random.default_rng(seed + B + H + C + Cout + k)
    x = g.integers(0, 4, (B, H, W, C), dtype=np.uint8)
    w = g.integers(0, 4, (Cout, k, k, C), dtype=np.uint8)
    pad = k // 2
    T = oracle.build_lut16(WL, AL)
    exp = oracle.conv2d_direct(x, w, T, stride, pad, 0).reshape(-1, Cout)
    xp = pack(x.reshape(-1, C))[:, : C // 4].contiguous()
    wp = pack(w.reshape(Cout, -1), True)
    w4 = dg.expand_operand_f4(wp, k * k * C, WL)
    p = dg.conv_params(B, H, W, C, Cout, k, k, stride, pad, 0, ldw=wp.shape[1])
    lut = dg.build_lut(WL, AL, 8)
    bias = (-int(np.round(exp.mean())) + g.integers(-30, 30, Cout)).astype(np.int32)
    rq = dg.Requant(20000, 20, 1, 0, 3, bias=torch.from_numpy(bias).to(DEV), bias_axis=0)
    with dg.options(**opts):
        out = dg.lut_conv2d_f4_prepared(xp, w4, lut, p)
        tag = dg.last_kernel()
        codes = dg.lut_conv2d_f4_prepared(xp, w4, lut, p, rq=rq)
    torch.cuda.synchronize()
    ok = np.array_equal(out.cpu().numpy(), exp) and np.array_equal(
        codes_of(codes, exp.shape[0], Cout), oracle.requantize(exp, 20000, 20, 1, 0, 3, bias=bias, bias_axis=0))
    return tag, ok


def onehot_case():
    g = np.random.default_rng(4)
    M, N, K = 130, 200, 300
    T = g.integers(-100, 101, 16).astype(np.int32)
    W = g.integers(0, 4, (M, K), dtype=np.uint8)
    A = g.integers(0, 4, (K, N), dtype=np.uint8)
    lut = dg.lut_from_table(T, 8)
    C = dg.lut_gemm_onehot(dg.expand_onehot(pack(W, True), K), dg.expand_tcols(pack(A.T), K, lut), M, N, K, lut)
    torch.cuda.synchronize()
    return dg.last_kernel(), np.array_equal(C.cpu().numpy(), oracle.lut_gemm(W, A, T))


def variant_case(variant):
    g = np.random.default_rng(5)
    M, N, K = 70, 150, 333
    W = g.integers(0, 4, (M, K), dtype=np.uint8)
    A = g.integers(0, 4, (K, N), dtype=np.uint8)
    lut = dg.build_lut(WL, AL, 8)
    C = dg.lut_gemm(pack(W, True), pack(A.T), M, N, K, lut, variant=variant)
    torch.cuda.synchronize()
    return dg.last_kernel(), np.array_equal(C.cpu().numpy(), oracle.lut_gemm(W, A, oracle.build_lut16(WL, AL)))


CASES = {
    "ts64_k128": lambda: gemm_case(300, 64, 64, {}),
    "ts64_k256": lambda: gemm_case(300, 64, 256, {}),
    "ts128_k128": lambda: gemm_case(300, 128, 128, {}),
    "ts128_k256s": lambda: gemm_case(300, 128, 256, {}),
    "asm": lambda: gemm_case(300, 256, 64, {}),
    "bn256": lambda: gemm_case(300, 256, 3200, {}),
    "ts128_long": lambda: gemm_case(300, 128, 1152, {}),
    "ts64_long": lambda: gemm_case(300, 64, 1152, {}),
    "ts128_kst128": lambda: gemm_case(300, 96, 1152, {"kst": 128}),
    "nobres_nof16": lambda: gemm_case(300, 128, 1152, {"bres": 0, "f16": 0}),
    "implicit_s2": lambda: conv_case(2, 9, 9, 64, 128, 3, 2, {}),
    "implicit_256": lambda: conv_case(1, 8, 8, 256, 256, 3, 1, {"win": -1}),
    "win64_pair": lambda: conv_case(2, 10, 10, 64, 64, 3, 1, {"win": 1}),
    "win64_res": lambda: conv_case(2, 10, 10, 64, 64, 3, 1, {"win": 1}, res=True),
    "win128_tile": lambda: conv_case(2, 9, 9, 128, 96, 3, 1, {"win": 1, "win128": 1}),
    "win128_kst256": lambda: conv_case(2, 9, 9, 128, 96, 3, 1, {"win": 1, "win128": 0}),
    "win256": lambda: conv_case(1, 7, 7, 256, 128, 3, 1, {"win": 1}),
    "splitk": lambda: conv_case(1, 7, 7, 256, 256, 3, 1, {"win": -1}, ws_fill=0xA5),
    "splitk_res": lambda: conv_case(1, 7, 7, 256, 128, 3, 1, {"win": -1}, ws_fill=0xA5, res=False),
    "direct_res": lambda: conv_case(2, 6, 6, 64, 64, 1, 1, {}, res=True),
    "f4": f4_case,
    "f4conv_bn256": lambda: f4conv_case(2, 9, 9, 256, 512, 1, 1, {}),
    "f4conv_bn256_e4": lambda: f4conv_case(2, 9, 9, 256, 256, 1, 1, {"f4_epi": 4, "f4_omma": 0}),
    "f4conv_bn128": lambda: f4conv_case(2, 9, 9, 256, 128, 1, 1, {}),
    "f4conv_bn64": lambda: f4conv_case(2, 9, 9, 256, 64, 1, 1, {}),
    "f4conv_gather": lambda: f4conv_case(1, 8, 8, 256, 256, 3, 1, {}),
    "f4conv_gather_s2": lambda: f4conv_case(2, 9, 9, 128, 128, 3, 2, {}),
    "f4conv_ct2": lambda: f4conv_case(2, 9, 9, 256, 128, 1, 1, {"f4_ct": 2}),
    "f4conv_win": lambda: f4conv_case(2, 10, 10, 64, 128, 3, 1, {"f4_win": 1}),
    "splitk_fused": lambda: conv_case(1, 7, 7, 256, 256, 3, 1, {"win": -1, "skfuse": 1}, ws_fill=0xA5),
    "onehot": onehot_case,
    "cc": lambda: variant_case("cc"),
    "tc_ss": lambda: variant_case("tc_ss"),
}


def main():
    sel = sys.argv[1:] or list(CASES)
    bad = 0
    for name in sel:
        tag, ok = CASES[name]()
        bad += not ok
        print(f"{name:16s} {'OK ' if ok else 'BAD'} {tag}", flush=True)
    print("ALL OK" if bad == 0 else f"{bad} BAD")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
