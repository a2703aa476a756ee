"""Run selected layers of a conv workload (for ncu / per-kernel timing)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2304_09049_b200 import netrun  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=3)
ap.add_argument("--layers", default="2")
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--variant", default="auto")
ap.add_argument("--no-rq", action="store_true")
a = ap.parse_args()
r = netrun.NetRunner(a.cfg, range(a.batch), "cuda", variant=a.variant, layers=[int(x) for x in a.layers.split(",")])
if a.no_rq:
    for p in r.plans:
        p.rq = None
        p.out = torch.empty((p.rows, p.layer.cout), dtype=torch.int32, device="cuda")
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in r.plans]
for i in range(a.iters):
    r.step(gemm_events=ev)
torch.cuda.synchronize()
for p, (e0, e1) in zip(r.plans, ev):
    ms = e0.elapsed_time(e1)
    print(f"{p.name}: rows={p.rows} cout={p.layer.cout} K={p.K} gemm {ms:.4f} ms  {p.ops / ms / 1e9:.1f} TOPS")
