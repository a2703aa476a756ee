import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2304_09049_b200 import dg
import oracle
WL, AL = [-2, -1, 0, 1], [0, 1, 2, 3]
lut = dg.build_lut(WL, AL, 8)
g = np.random.default_rng(0)
for (M, N, K, rqon) in [(64, 16, 144, False), (64, 16, 144, True), (300, 96, 64, False), (300, 96, 64, True), (64, 64, 576, True)]:
    A = g.integers(0, 4, (M, K), dtype=np.uint8)
    Wt = g.integers(0, 4, (N, K), dtype=np.uint8)
    a_p = dg.pack_codes(torch.from_numpy(A).cuda())
    w_p = dg.pack_codes(torch.from_numpy(Wt).cuda())
    w8 = dg.expand_operand(w_p, K, WL)
    lut_t = dg.build_lut(AL, WL, 8)
    rq = dg.Requant(30000, 20, 1, 0, 3, bias=torch.full((N,), 3, dtype=torch.int32, device="cuda"), bias_axis=0) if rqon else None
    try:
        out = dg.lut_gemm_prepared(a_p, w8, M, N, K, lut_t, rq=rq)
        torch.cuda.synchronize()
        print(M, N, K, rqon, "ok", flush=True)
    except Exception as e:
        print(M, N, K, rqon, "FAIL", e, flush=True)
        break
