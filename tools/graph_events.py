"""Does recording external CUDA events around every layer inside the captured step graph cost time
(e.g. by breaking programmatic-dependent-launch overlap between layers)?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2304_09049_b200 import netrun
r = netrun.NetRunner(3, range(256), "cuda")
for _ in range(3):
    r.step()
torch.cuda.synchronize()
nl = len(r.plans)
gev = [(torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True)) for _ in range(nl)]
g_ev, g_plain = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
with torch.cuda.graph(g_ev):
    r.step(gemm_events=gev)
with torch.cuda.graph(g_plain):
    r.step()
for g in (g_ev, g_plain, g_ev, g_plain):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(30):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print("events" if g is g_ev else "plain ", f"{e0.elapsed_time(e1) / 30:.4f} ms/step")
