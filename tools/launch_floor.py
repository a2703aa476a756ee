"""Latency floor of one dependent launch of the tensor-core GEMM kernel: a CUDA graph of back-to-back
tiny GEMMs (one 128x64 tile, K = 64) with and without programmatic dependent launch, and a chain
of 19 launches shaped like the ResNet-18 b1 convs' critical paths (config 2's latency budget)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2304_09049_b200 import dg  # noqa: E402

lut = dg.build_lut([0, 1, 2, 3], [-2, -1, 0, 1], 8)


def floor(M, N, K, n=30, pdl=1):
    dg.set_option("pdl", pdl)
    ld = dg.packed_ld(K)
    a = torch.randint(0, 256, (M, ld), dtype=torch.uint8, device="cuda")
    w8 = dg.expand_operand(torch.randint(0, 256, (N, ld), dtype=torch.uint8, device="cuda"), K, [-2, -1, 0, 1])
    out = torch.empty((M, N), dtype=torch.int32, device="cuda")
    dg.lut_gemm_prepared(a, w8, M, N, K, lut, out=out)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            dg.lut_gemm_prepared(a, w8, M, N, K, lut, out=out)
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / n)
    return sorted(ts)[3]


for pdl in (1, 0):
    print(f"pdl={pdl}: 128x64x64 (one tile): {floor(128, 64, 64, pdl=pdl):6.2f} us/launch;  "
          f"128x512x4608 (one tile row, 36 stages): {floor(128, 512, 4608, pdl=pdl):6.2f} us/launch", flush=True)
