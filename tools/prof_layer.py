"""Time selected layers of a conv workload per dg option setting (for A/B of kernel instances).

  python tools/prof_layer.py --cfg 3 --layers 2,3,12 --sweep em=0,1,2,3 [--opt early_weights=1]

Each layer is timed alone (CUDA events around its launch, median of --iters replays of a CUDA graph
holding --reps back-to-back launches of that layer, so the PDL prologue overlap is included), and
the instance tag (dg_last_kernel) is printed.  Codes of every setting are compared with the first
setting's (all settings must give identical outputs)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2304_09049_b200 import dg, netrun  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=3)
ap.add_argument("--layers", default="2")
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--reps", type=int, default=8)
ap.add_argument("--opt", action="append", default=[])
ap.add_argument("--sweep", default="")
ap.add_argument("--f4", default="", help="comma-separated layer ids on the FP4 conv kernel ('all' = every layer given, "
                                         "'default' = netrun.f4_default's routing; empty = int8 kernels only)")
a = ap.parse_args()
for o in a.opt:
    k, v = o.split("=")
    dg.set_option(k, int(v))
batch = a.batch or (256 if a.cfg == 3 else 64)
layers = [int(x) for x in a.layers.split(",")]
f4 = set() if not a.f4 else (None if a.f4 == "default" else (set(layers) if a.f4 == "all" else {int(x) for x in a.f4.split(",")}))
r = netrun.NetRunner(a.cfg, range(batch), "cuda", layers=layers, f4=f4)
sweep = [("", [None])]
if a.sweep:
    k, vs = a.sweep.split("=")
    sweep = [(k, [int(v) for v in vs.split(",")])]
ref = None
for key, vals in sweep:
    for v in vals:
        if key:
            dg.set_option(key, v)
        outs = []
        total = 0.0
        for i, p in enumerate(r.plans):
            sub = netrun.NetRunner.__new__(netrun.NetRunner)
            sub.__dict__.update(r.__dict__)
            sub.plans = [p]
            sub.step()
            tag = p.kernel
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(a.reps):
                    sub.step()
            ts = []
            for _ in range(a.iters):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / a.reps)
            ms = sorted(ts)[len(ts) // 2]
            outs.append(p.out.clone())
            total += ms * 1e3
            print(f"{key}={v} L{layers[i]:02d} {p.name:24s} rows={p.rows} cout={p.layer.cout} K={p.K} "
                  f"{ms * 1e3:7.1f} us {p.ops / ms / 1e9:7.1f} TOPS  [{tag}]", flush=True)
        print(f"{key}={v}: sum over the layers {total:.1f} us", flush=True)
        if ref is None:
            ref = outs
        else:
            same = all(torch.equal(x, y) for x, y in zip(ref, outs))
            print(f"{key}={v}: outputs {'identical' if same else 'DIFFER'} to the first setting", flush=True)
