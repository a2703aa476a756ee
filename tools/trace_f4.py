"""CTA-0 event timeline of the FP4 conv kernel (needs libdg_trace.so, built with -DDG_TRACE).
usage: python tools/trace_f4.py LAYER [--cfg 3] [--opt name=value ...]
Per stage g: 0 B TMA issued, 12 unpack P ready, 13 unpack empty_a ok, 5 unpack full_a arrive,
2 waiter full_a ok, 3 waiter full_b ok, 14 MMA warp past the hand-off, 15 MMAs issued,
4 commits issued.  Per tile t: 1 waiter acc_empty ok,
6/9 epi group 0/1 acc_full ok, 7/10 released, 8/11 done (cycles from the first event)."""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["DG_LIB_PATH"] = os.path.join(ROOT, "paper_2304_09049_b200", "libdg_trace.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2304_09049_b200 import dg, netrun  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("layer", type=int)
ap.add_argument("--cfg", type=int, default=3)
ap.add_argument("--opt", action="append", default=[])
ap.add_argument("--n", type=int, default=40)
a = ap.parse_args()
for o in a.opt:
    k, v = o.split("=")
    dg.set_option(k, int(v))
r = netrun.NetRunner(a.cfg, range(256 if a.cfg == 3 else 64), "cuda", layers=[a.layer], f4={a.layer})
L = dg.lib()
TN, TE = 96, 16
buf = (ctypes.c_longlong * (TE * TN))()
for it in range(2):
    L.dg_debug_cf_timeline(buf, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r.step()
    e1.record()
    torch.cuda.synchronize()
L.dg_debug_cf_timeline(buf, 0)
t = np.frombuffer(buf, dtype=np.int64).reshape(TE, TN).astype(np.int64)
print(f"L{a.layer} {r.plans[0].name}: {e0.elapsed_time(e1) * 1e3:.1f} us  [{r.plans[0].kernel}]")
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, -1)
print("stage   B_tma  unp_P  unp_eA unp_fA  w_fA   w_fB  m_hoff  m_iss  m_com")
for g in range(a.n):
    print(f"{g:5d} " + " ".join(f"{t[e][g]:6d}" for e in (0, 12, 13, 5, 2, 3, 14, 15, 4)))
print("tile  w_accE  e0_full e0_rel e0_done e1_full e1_rel e1_done")
for i in range(a.n):
    print(f"{i:4d} " + " ".join(f"{t[e][i]:7d}" for e in (1, 6, 7, 8, 9, 10, 11)))
