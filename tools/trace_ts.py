"""CTA-0 event timeline of the TS kernel (needs libdg_trace.so, built with -DDG_TRACE).
usage: python tools/trace_ts.py MxNxK [--rq]      (P = M rows unpacked into TMEM, N = weight rows)
Events per stage g / tile t (cycles, clock64 of SM 0):
  12 producer issued P TMA(g)   0 unpack start(g)  1 unpack data ready(g)  11 empty_a ok(g)  2 full_a arrive(g)
   3 waiter start tile(t)       4 waiter full_a ok(g)  5 waiter full_b ok(g)  6 MMA start(g)  7 MMA issued(g)
   8 epi start(t)  9 epi acc_full ok(t)  10 epi done(t)"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["DG_LIB_PATH"] = os.path.join(ROOT, "paper_2304_09049_b200", os.environ.get("DG_TRACE_LIB", "libdg_trace.so"))
import numpy as np
import torch
from paper_2304_09049_b200 import dg
CONV = sys.argv[1].startswith("conv") if len(sys.argv) > 1 else False   # conv<layer>: ResNet-50 layer via netrun
M, N, K = (1, 1, 1) if CONV else map(int, (sys.argv[1] if len(sys.argv) > 1 else "802816x64x64").split("x"))
lut = dg.build_lut([0, 1, 2, 3], [-2, -1, 0, 1], 8)
if CONV:
    from paper_2304_09049_b200 import netrun
    cfg = int(os.environ.get("DG_TRACE_CFG", "3"))   # 3: ResNet-50 b256, 4: VGG-16 b64
    runner = netrun.NetRunner(cfg, range(256 if cfg == 3 else 64), "cuda", layers=[int(sys.argv[1][4:])])
    M, N, K = runner.plans[0].rows, runner.plans[0].layer.cout, runner.plans[0].K
ld = dg.packed_ld(K)
w = torch.randint(0, 256, (M, ld), dtype=torch.uint8, device="cuda")
at = torch.randint(0, 256, (N, ld), dtype=torch.uint8, device="cuda")
at8 = dg.expand_operand(at, K, lut.al)
if "--rq" in sys.argv:
    out = torch.empty((M, N // 4), dtype=torch.uint8, device="cuda")
    rq = dg.Requant(30000, 20, 0, 0, 3, bias=torch.full((N,), K // 2, dtype=torch.int32, device="cuda"), bias_axis=0)
else:
    out = torch.empty((M, N), dtype=torch.int32, device="cuda")
    rq = None
L = dg.lib()
TLN = 96
TLE = 24
buf = (ctypes.c_longlong * (TLE * TLN))()
for it in range(2):
    L.dg_debug_ts_timeline(buf, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if CONV:
        runner.step()
    else:
        dg.lut_gemm_prepared(w, at8, M, N, K, lut, rq=rq, out=out)
    e1.record(); torch.cuda.synchronize()
L.dg_debug_ts_timeline(buf, 0)
a = np.frombuffer(buf, dtype=np.int64).reshape(TLE, TLN).astype(np.int64)
print(f"{M}x{N}x{K}: {e0.elapsed_time(e1):.3f} ms")
t0 = a[a > 0].min()
a = np.where(a > 0, a - t0, -1)
nst = (K + 127) // 128
names = {13: "P_loop", 12: "P_tma", 0: "unp0", 20: "P_ok", 21: "unp_alu", 1: "unp_rdy", 11: "emptyA", 2: "fullA", 4: "w_fullA", 5: "w_fullB", 6: "handoff"}
print("stage " + " ".join(f"{v:>8s}" for v in names.values()))
for g in list(range(0, int(os.environ.get('TRACE_STAGES', '40')))):
    print(f"{g:5d} " + " ".join(f"{a[e][g]:8d}" for e in names))
if "--prod" in sys.argv:
    print("stage  work_item  P_loop  wait_ok  issued  synced   (producer warp)")
    for g in range(0, 40):
        print(f"{g:5d} " + " ".join(f"{a[e][g]:8d}" for e in (23, 13, 14, 12, 22)))
if len(sys.argv) > 2 and sys.argv[2] == "--short":
    print("tile  P_loop P_tma unp0 unp_done w_start w_fullA handoff epi0 epi_accfull epi_done")
    for t in range(0, 40):
        print(f"{t:4d} " + " ".join(f"{a[e][t]:8d}" for e in (13, 12, 0, 2, 3, 4, 6, 8, 9, 10)))
if len(sys.argv) > 2 and sys.argv[2] == "--win":
    print("stage: waiter_fullA w_fullB handoff mma_prebar mma_bar mma_start mma_end")
    for g in range(0, 30):
        print(f"{g:4d} " + " ".join(f"{a[e][g]:8d}" for e in (4, 5, 6, 13, 7, 14, 15)))
    print("tile unp0 cpa_ok unpacked fetched emptyW fullW_arr waiter_fullW  w_start epi0 epi_accfull epi_done")
    for t in range(0, 40):
        print(f"{t:4d} " + " ".join(f"{a[e][t]:8d}" for e in (0, 12, 21, 1, 11, 2, 13, 3, 8, 9, 10)))
print("tile  w_start  epi0   epi_accfull  ld0_ok  r0_done  ld1_ok  r1_done  epi_done   (warp 0: even tiles)")
for t in list(range(0, 16)) + list(range(38, 43)):
    print(f"{t:4d} " + " ".join(f"{a[e][t]:8d}" for e in (3, 8, 9, 16, 17, 18, 19, 10)))
