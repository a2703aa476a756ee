"""Time the conv-orientation GEMM (P = pixels) of a short-K 1x1 layer shape for several K (the
per-tile MMA count): separates accumulator traffic from the fixed per-tile epilogue cost."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2304_09049_b200 import dg  # noqa: E402

M = int(os.environ.get("KS_M", 802816))
N = int(os.environ.get("KS_N", 256))
dg.set_option("early_weights", 1)
lut_t = dg.build_lut([0, 1, 2, 3], [-2, -1, 0, 1], 8)
for K in [int(x) for x in os.environ.get("KS_K", "32,64,96,128,192,256").split(",")]:
    ld = dg.packed_ld(K)
    a = torch.randint(0, 256, (M, ld), dtype=torch.uint8, device="cuda")
    if K % 64:
        a[:, K // 4:] = 0
    w = torch.randint(0, 256, (N, ld), dtype=torch.uint8, device="cuda")
    w8 = dg.expand_operand(w, K, [-2, -1, 0, 1])
    out = torch.empty((M, N // 4), dtype=torch.uint8, device="cuda")
    rq = dg.Requant(30000, 20, 0, 0, 3, bias=torch.full((N,), -K // 3, dtype=torch.int32, device="cuda"))
    for mode in ("codes", "int32"):
        o = out if mode == "codes" else torch.empty((M, N), dtype=torch.int32, device="cuda")
        r = rq if mode == "codes" else None
        dg.lut_gemm_prepared(a, w8, M, N, K, lut_t, rq=r, out=o)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(8):
                dg.lut_gemm_prepared(a, w8, M, N, K, lut_t, rq=r, out=o)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 8)
        print(f"M={M} N={N} K={K:4d} {mode:5s}: {sorted(ts)[2] * 1e3:7.1f} us  [{dg.last_kernel()[:60]}]", flush=True)
