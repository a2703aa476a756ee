"""Per-conv GPU time of the ResNet-18 b1 chain (config 2), eager, CUDA events around each call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2304_09049_b200 import netrun  # noqa: E402

r = netrun.ResNet18Runner("cuda", batch=int(sys.argv[1]) if len(sys.argv) > 1 else 1)
orig = r._conv
ev = []


def timed(x, li, rq, out, stream):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    orig(x, li, rq, out, stream)
    b.record()
    ev.append((li, a, b))


r._conv = timed
for _ in range(3):
    ev.clear()
    r.step()
torch.cuda.synchronize()
tot = 0.0
for li, a, b in ev:
    L = r.layers[li]
    ms = a.elapsed_time(b)
    tot += ms
    print(f"conv{li:2d} {L.cin:4d}->{L.cout:4d} k{L.k} s{L.stride} {L.h:3d}x{L.h:<3d} rows={L.ho * L.ho * r.B:6d} K={L.K:5d}  {ms * 1e3:7.1f} us")
print(f"total {tot * 1e3:.1f} us")
