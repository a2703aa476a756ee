import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2304_09049_b200 import dg
import synth
WL, AL = [-2, -1, 0, 1], [0, 1, 2, 3]
lut = dg.build_lut(WL, AL, 8)
W = synth.uniform_codes((64, 576), 1, 0, synth.T_W)
A = synth.uniform_codes((576, 196), 1, 0, synth.T_A)
w = dg.pack_codes(torch.from_numpy(W).cuda(), weights=True)
at = dg.pack_codes(torch.from_numpy(np.ascontiguousarray(A.T)).cuda())
dg.lut_gemm(w, at, 64, 196, 576, lut, variant="tc_ss"); torch.cuda.synchronize(); print("ss ok", flush=True)
z = dg.pack_codes(torch.zeros((1, 4), dtype=torch.uint8, device="cuda"))
dg.lut_gemm(z, z, 1, 1, 4, lut, variant="tc"); torch.cuda.synchronize(); print("probe ok", flush=True)
