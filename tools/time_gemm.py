"""Quick CUDA-event timing of dg_lut_gemm variants on synthetic square / conv-like shapes."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2304_09049_b200 import dg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="4096x4096x4096,8192x8192x8192,802816x64x576,50176x256x2304")
ap.add_argument("--variants", default="cc,tc,tc_ss,prepared")
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
lut = dg.build_lut([-2, -1, 0, 1], [0, 1, 2, 3], 8)
for s in a.shapes.split(","):
    M, N, K = map(int, s.split("x"))
    ld = dg.packed_ld(K)
    w = torch.randint(0, 256, (M, ld), dtype=torch.uint8, device="cuda")
    at = torch.randint(0, 256, (N, ld), dtype=torch.uint8, device="cuda")
    out = torch.empty((M, N), dtype=torch.int32, device="cuda")
    ws = torch.empty(dg.gemm_workspace_size(M, N, ld * 4), dtype=torch.uint8, device="cuda")
    at8 = dg.expand_operand(at, ld * 4, lut.al)
    for v in a.variants.split(","):
        if v == "cc" and M * N * K > 2 ** 36:
            continue
        if v == "prepared":
            f = lambda: dg.lut_gemm_prepared(w, at8, M, N, ld * 4, lut, out=out)
        elif v == "onehot":   # any int8 table on the tensor cores (K' = 4K)
            w1h = dg.expand_onehot(w, ld * 4)
            atc = dg.expand_tcols(at, ld * 4, lut)
            f = lambda: dg.lut_gemm_onehot(w1h, atc, M, N, ld * 4, lut, out=out)
        elif v == "gemm4":   # 4-bit codes (the same random bytes read as 2 codes each), K4 = 2 * ld
            lv16 = [((i * 7) % 31) - 15 for i in range(16)]
            w8d = dg.expand_digits4(w, ld * 2, lv16)
            out4 = torch.empty((N, M), dtype=torch.int32, device="cuda")
            f = lambda: dg.lut_gemm4_prepared(at, w8d, N, M, ld * 2, lv16, out=out4)
        elif v == "f4":   # block-scaled FP4 path: weights expanded once to e2m1
            w4 = dg.expand_operand_f4(w, ld * 4, lut.wl)
            f = lambda: dg.lut_gemm_f4(w4, at, M, N, ld * 4, lut, out=out)
        else:
            f = lambda: dg.lut_gemm(w, at, M, N, ld * 4, lut, variant=v, out=out, ws=ws)
        try:
            f()
        except dg.DGError as e:
            print(f"{s} {v}: {e}")
            continue
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        ops = 2 * M * N * ld * (2 if v == "gemm4" else 4)   # (4-bit: K = 2 codes per byte)
        print(f"{s} {v}: {ms:.3f} ms  {ops / ms / 1e9:.1f} TOPS")
