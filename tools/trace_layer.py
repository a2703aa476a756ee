"""Pipeline timeline of the tc kernel for CTA 0 (needs libdg_trace.so built with -DDG_TRACE)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["DG_LIB_PATH"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2304_09049_b200", "libdg_trace.so")
import torch
from paper_2304_09049_b200 import dg, netrun
layer = int(sys.argv[1]) if len(sys.argv) > 1 else 0
r = netrun.NetRunner(3, range(256), "cuda", layers=[layer])
buf = torch.zeros(11 * 64, dtype=torch.int64, device="cuda")
r.step(); torch.cuda.synchronize()
dg.lib().dg_debug_set_trace(ctypes.c_void_p(buf.data_ptr()))
r.step(); torch.cuda.synchronize()
t = buf.view(11, 64).cpu().numpy()
t0 = t[0, 0]
names = ["tma_slot_free", "mma_acc_free", "mma_full_u", "unp_full_p", "unp_empty_u", "unp_done", "epi_acc_full", "epi_released", "epi_stored", "unp_loop_end", "unp_fenced"]
for i in range(16):
    print(i, " ".join(f"{n}={(t[k, i] - t0) / 1000:8.2f}" for k, n in enumerate(names) if t[k, i]))
