import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2304_09049_b200 import dg
WL, AL = [-2, -1, 0, 1], [0, 1, 2, 3]
lut = dg.build_lut(WL, AL, 8)
for shape in [(1, 1, 4), (1, 1, 64), (2, 3, 4), (1, 16, 4), (1, 32, 4), (1, 64, 4), (1, 65, 4), (1, 256, 4), (1, 1, 4)]:
    M, N, K = shape
    w = dg.pack_codes(torch.zeros((max(M, N), K), dtype=torch.uint8, device="cuda"))
    try:
        dg.lut_gemm(w[:M], w[:N], M, N, K, lut, variant="tc")
        torch.cuda.synchronize()
        print(shape, "ok", flush=True)
    except Exception as e:
        print(shape, "FAIL", str(e)[:100], flush=True)
        break
