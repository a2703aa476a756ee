"""Cycle breakdown of the TS kernel's MMA issue loop (CTA 0), needs libdg_trace.so."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["DG_LIB_PATH"] = os.path.join(ROOT, "paper_2304_09049_b200", os.environ.get("DG_TRACE_LIB", "libdg_trace.so"))
import torch
from paper_2304_09049_b200 import dg
M, N, K = map(int, (sys.argv[1] if len(sys.argv) > 1 else "8192x8192x8192").split("x"))
lut = dg.build_lut([-2, -1, 0, 1], [0, 1, 2, 3], 8)
ld = dg.packed_ld(K)
w = torch.randint(0, 256, (M, ld), dtype=torch.uint8, device="cuda")
at = torch.randint(0, 256, (N, ld), dtype=torch.uint8, device="cuda")
at8 = dg.expand_operand(at, K, lut.al)
RQ = "--rq" in sys.argv
if RQ:
    out = torch.empty((M, N // 4), dtype=torch.uint8, device="cuda")
    bias = torch.full((N,), K // 2, dtype=torch.int32, device="cuda")
    rq = dg.Requant(30000, 20, 0, 0, 3, bias=bias, bias_axis=0)
else:
    out = torch.empty((M, N), dtype=torch.int32, device="cuda")
    rq = None
L = dg.lib()
buf = (ctypes.c_ulonglong * 16)()
dg.lut_gemm_prepared(w, at8, M, N, K, lut, rq=rq, out=out); torch.cuda.synchronize()
L.dg_debug_ts_prof(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); dg.lut_gemm_prepared(w, at8, M, N, K, lut, rq=rq, out=out); e1.record(); torch.cuda.synchronize()
L.dg_debug_ts_prof(buf, 0)
n = buf[3]
ntile = max(buf[11], 1)
ns = max(buf[13], 1)
print(f"  unpack stage: load(+wait full_p)={buf[6]/ns:.0f} unpack={buf[7]/ns:.0f} wait_empty_a={buf[10]/ns:.0f} tmem_st+wait={buf[14]/ns:.0f}")
print(f"  epilogue warp0: wait_acc={buf[8]/ntile:.0f} work={buf[9]/ntile:.0f} cycles/tile over {ntile} tiles; unpack warp: {buf[12]/max(buf[13],1):.0f} cycles/stage")
print(f"{M}x{N}x{K}: {e0.elapsed_time(e1):.3f} ms; CTA0 stages={n}  mma_barsync={buf[0]/n:.0f}  mma_issue={buf[2]/n:.0f}  waiter_full_a={buf[4]/n:.0f} waiter_full_b={buf[5]/n:.0f} cycles/stage")
