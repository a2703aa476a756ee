import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2304_09049_b200 import dg
import oracle
WL, AL = [-2, -1, 0, 1], [0, 1, 2, 3]
lut_t = dg.build_lut(AL, WL, 8)
g = np.random.default_rng(0)
for (M, N, K) in [(300, 64, 64), (300, 64, 256), (300, 64, 1024), (300, 256, 64), (5000, 64, 64)]:
    A = g.integers(0, 4, (M, K), dtype=np.uint8)
    Wt = g.integers(0, 4, (N, K), dtype=np.uint8)
    a_p = dg.pack_codes(torch.from_numpy(A).cuda())
    w_p = dg.pack_codes(torch.from_numpy(Wt).cuda())
    w8 = dg.expand_operand(w_p, K, WL)
    try:
        out = dg.lut_gemm_prepared(a_p, w8, M, N, K, lut_t)
        torch.cuda.synchronize()
        exp = oracle.lut_gemm(A, np.ascontiguousarray(Wt.T), oracle.build_lut16(AL, WL))
        print(M, N, K, "ok", np.array_equal(out.cpu().numpy(), exp), flush=True)
    except Exception as e:
        print(M, N, K, "FAIL", str(e)[:80], flush=True)
        break
