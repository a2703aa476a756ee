"""Calibrate config 2's per-layer requant parameters (reading Q12/Q13) on the synthetic input,
running ONLY the CPU oracle chain (like post-training-quantisation calibration).  Writes
synth_data/resnet18_requant.json, read by synth.resnet18_requants().

For every conv the parameters centre its pre-requant value v = acc + residual:
    bias = -round(mean(v)),  mult = round(2^20 * 1.5 / std(v)),  shift 20, zp 0, codes 0..3
and identity residuals use res_mult = round(0.5 * std(acc) / std(al[x])).
These are inputs of the computation (config data), not expected outputs."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2304_09049_b200 import netrun  # noqa: E402  (input generators only)


def main():
    L = synth.resnet18_layers()
    T = oracle.build_lut16(synth.WL_UNIFORM, synth.AL_UNIFORM)
    al = np.array(synth.AL_UNIFORM, np.int64)
    x = netrun.input_codes(2, 0, L[0], [0], "cpu").numpy()
    out = {}
    gain = 1.5
    for c1, c2, ds in synth.resnet18_blocks():
        W = {li: netrun.weight_codes(2, li, L[li], "cpu").numpy() for li in (c1, c2) + ((ds,) if ds is not None else ())}
        a1 = oracle.conv2d_direct(x, W[c1], T, L[c1].stride, L[c1].pad, 0).reshape(-1, L[c1].cout).astype(np.int64)
        m1 = int(round(2 ** 20 * gain / a1.std()))
        b1 = -int(round(a1.mean()))
        out[c1] = {"mult": m1, "shift": 20, "zp": 0, "bias": b1, "res_mult": 0}
        y1 = oracle.requantize(a1.astype(np.int32), m1, 20, 0, 0, 3, bias=np.full(L[c1].cout, b1, np.int32))
        y1 = y1.reshape(1, L[c1].ho, L[c1].ho, L[c1].cout)
        a2 = oracle.conv2d_direct(y1, W[c2], T, L[c2].stride, L[c2].pad, 0).reshape(-1, L[c2].cout).astype(np.int64)
        if ds is not None:
            res = oracle.conv2d_direct(x, W[ds], T, L[ds].stride, L[ds].pad, 0).reshape(-1, L[ds].cout).astype(np.int64)
            rm = 0
            out[ds] = {"mult": 0, "shift": 20, "zp": 0, "bias": 0, "res_mult": 0}
        else:
            lv = al[x.reshape(-1, L[c2].cout)]
            rm = max(1, int(round(0.5 * a2.std() / max(lv.std(), 1e-9))))
            res = lv * rm
        v = a2 + res
        m2 = int(round(2 ** 20 * gain / v.std()))
        b2 = -int(round(v.mean()))
        out[c2] = {"mult": m2, "shift": 20, "zp": 0, "bias": b2, "res_mult": rm}
        o = oracle.requantize(a2.astype(np.int32), m2, 20, 0, 0, 3, res=res.astype(np.int32),
                              bias=np.full(L[c2].cout, b2, np.int32))
        x = o.reshape(1, L[c2].ho, L[c2].ho, L[c2].cout)
        print(f"block {c1}: out code histogram {np.round(np.bincount(o.ravel(), minlength=4) / o.size, 3)}")
    path = os.path.join(ROOT, "synth_data", "resnet18_requant.json")
    with open(path, "w") as f:
        json.dump({"source": "tools/calibrate_resnet18.py (oracle chain only)", "layers": {str(k): v for k, v in sorted(out.items())}}, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
