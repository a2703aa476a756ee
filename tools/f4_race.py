"""Reproduce / bisect nondeterminism of the FP4 conv kernel on one full-batch ResNet-50 layer:
run the layer's int32 step N times under option settings and report how many outputs differ from
the first run and from the oracle's whole-output Freivalds check."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2304_09049_b200 import dg, netrun  # noqa: E402

li = int(sys.argv[1]) if len(sys.argv) > 1 else 10
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
L = synth.resnet50_layers()[li]
T = oracle.build_lut16(synth.WL_UNIFORM, synth.AL_UNIFORM)
x = synth.counter_codes_host(0, 256 * L.h * L.h * L.cin, (3, li, synth.T_X), "relu").reshape(256, L.h, L.h, L.cin)
w = synth.counter_codes_host(0, L.cout * L.k * L.k * L.cin, (3, li, synth.T_W), "uniform").reshape(L.cout, L.k, L.k, L.cin)
for opts in [dict(), dict(f4_unp=8)][: int(os.environ.get('NOPTS', '2'))]:
    dg.reset_options()
    for k, v in opts.items():
        dg.set_option(k, v)
    r = netrun.NetRunner(3, range(256), "cuda", layers=[li], f4={li})
    acc = r.int32_buffers()
    first = None
    ndiff, nbad = 0, 0
    for i in range(reps):
        acc[0].fill_(-7)
        r.step(int32_out=acc)
        torch.cuda.synchronize()
        a = acc[0].cpu().numpy()
        if first is None:
            first = a
        else:
            ndiff += int((a != first).sum())
        if i < 2:
            nbad += oracle.conv_freivalds(x, w, T, L.stride, L.pad, 0, a, seed=i)
    diffrows = np.unique(np.nonzero(a != first)[0]) if ndiff else []
    print(f"{opts}: {r.plans[0].kernel}: elements differing from run 0 over {reps} runs: {ndiff}; "
          f"Freivalds bad channels (2 runs): {nbad}; first differing rows {list(diffrows[:8])}", flush=True)
