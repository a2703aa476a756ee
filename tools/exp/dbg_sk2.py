import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2304_09049_b200 import dg
import oracle
WL, AL = [-2, -1, 0, 1], [0, 1, 2, 3]
lut = dg.build_lut(WL, AL, 8)
T = oracle.build_lut16(WL, AL)
g = np.random.default_rng(1)
def run(B, H, C, Cout, k, stride, prepared=True, iters=20):
    pad = k // 2
    x = g.integers(0, 4, (B, H, H, C), dtype=np.uint8)
    w = g.integers(0, 4, (Cout, k, k, C), dtype=np.uint8)
    exp = oracle.conv2d_direct(x, w, T, stride, pad, 0)
    xp = dg.pack_codes(torch.from_numpy(x.reshape(-1, C)).cuda())[:, :C // 4].contiguous()
    wp = dg.pack_codes(torch.from_numpy(w.reshape(Cout, -1)).cuda())
    w8 = dg.expand_operand(wp, k * k * C, WL)
    p = dg.conv_params(B, H, H, C, Cout, k, k, stride, pad, 0, ldw=wp.shape[1])
    ws = torch.zeros(dg.conv_workspace_size(p), dtype=torch.uint8, device="cuda")
    f = (lambda: dg.lut_conv2d_prepared(xp, w8, lut, p, ws=ws)) if prepared else (lambda: dg.lut_conv2d(xp, wp, lut, p, ws=ws))
    out = f(); torch.cuda.synchronize()
    ok = np.array_equal(out.cpu().numpy().reshape(exp.shape), exp)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): f()
    e1.record(); torch.cuda.synchronize()
    print(B, H, C, Cout, k, stride, "prepared" if prepared else "conv2d", "ok" if ok else "BAD", f"{e0.elapsed_time(e1) / iters * 1e3:.1f} us", flush=True)
run(3, 14, 128, 64, 3, 1, prepared=False)
run(3, 14, 128, 64, 3, 1, prepared=True)
run(1, 28, 128, 128, 3, 1)
run(1, 7, 512, 512, 3, 1)
os.environ["DG_NO_SPLITK"] = "1"
run(1, 28, 128, 128, 3, 1)
run(1, 7, 512, 512, 3, 1)
