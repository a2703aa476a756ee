"""GPU parity at BASELINE.json's full configuration sizes, in the launch configuration bench.py
times (netrun.NetRunner: every layer of the network back to back in ONE CUDA graph, programmatic
dependent launch, weights declared set-up data with the early_weights option, exactly as bench.py
runs the step).  All bit-exact:

  * every layer's WHOLE int32 output at full batch (ResNet-50 b256, VGG-16 b64) passes the
    oracle's exact conv Freivalds check (oracle.conv_freivalds: nonzero pixel weights, so any
    single wrong accumulator is caught), computed from host-drawn inputs (synth_gen.c);
  * every layer's requantised codes equal the oracle's direct conv + requant on 4 images spread
    across the batch (first, two interior, last);
  * the kernel instance each layer ran (dg_last_kernel) is recorded, and the default-dispatch
    instances the bench relies on all appear.
Inputs on both sides come from the same seeded counter generator (synth.py); expected values come
only from oracle/."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import synth  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2304_09049_b200 import dg, netrun  # noqa: E402

T_CONV = oracle.build_lut16(synth.WL_UNIFORM, synth.AL_UNIFORM)


def host_input(cfg, li, L, b0, nb):
    """NHWC codes of images [b0, b0+nb) of layer li, drawn on the host (same generator as netrun)."""
    per = L.h * L.h * L.cin
    return synth.counter_codes_host(b0 * per, nb * per, (cfg, li, synth.T_X), "relu").reshape(nb, L.h, L.h, L.cin)


def host_weights(cfg, li, L):
    n = L.cout * L.k * L.k * L.cin
    return synth.counter_codes_host(0, n, (cfg, li, synth.T_W), "uniform").reshape(L.cout, L.k, L.k, L.cin)


def oracle_codes(x1, w, L):
    acc = oracle.conv2d_direct(x1, w, T_CONV, L.stride, L.pad, 0)
    r = synth.conv_requant(L)
    return oracle.requantize(acc.reshape(-1, L.cout), r.mult, r.shift, r.zp, r.qmin, r.qmax,
                             bias=np.full(L.cout, r.bias, np.int32), bias_axis=0)


def run_graphs(r):
    """Capture the step (codes) and the int32 step in CUDA graphs like bench.py and replay them."""
    acc = r.int32_buffers()
    for _ in range(2):   # eager warm-up (sets kernel attributes), records the kernel tags
        r.step()
        r.step(int32_out=acc)
    g_codes, g_acc = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_codes):
        r.step()
    with torch.cuda.graph(g_acc):
        r.step(int32_out=acc)
    first = None
    for rep in range(3):   # every replay must reproduce the first bit for bit (a launch race would not)
        for p in r.plans:
            p.out.fill_(0xA5)
        for a in acc:
            a.fill_(-12345)
        g_codes.replay()
        g_acc.replay()
        torch.cuda.synchronize()
        if first is None:
            first = [p.out.clone() for p in r.plans] + [a.clone() for a in acc]
        else:
            now = [p.out for p in r.plans] + list(acc)
            diff = [i for i, (x, y) in enumerate(zip(first, now)) if not torch.equal(x, y)]
            assert not diff, ("replay differs", rep, [r.plans[i % len(r.plans)].kernel for i in diff])
    return acc


def check_network(cfg, batch, images):
    all_layers = synth.CONFIG_LAYERS[cfg]()
    with dg.options(early_weights=1):
        r = netrun.NetRunner(cfg, range(batch), "cuda")
        acc = run_graphs(r)
    kernels = {}
    pool = ThreadPoolExecutor(max_workers=8)   # (the oracle's ctypes calls release the GIL)
    for i, (plan, li) in enumerate(zip(r.plans, r.layer_ids)):
        L = all_layers[li]
        kernels[L.name] = plan.kernel
        x = host_input(cfg, li, L, 0, batch)
        w = host_weights(cfg, li, L)
        a = acc[i].cpu().numpy()
        codes_g = plan.out.cpu().numpy()
        rows = L.ho * L.ho
        futs = [pool.submit(oracle_codes, x[b:b + 1], w, L) for b in images]
        bad = oracle.conv_freivalds(x, w, T_CONV, L.stride, L.pad, 0, a, seed=li)
        assert bad == 0, (L.name, plan.kernel, "whole-output Freivalds", bad)
        for b, f in zip(images, futs):
            got = oracle.unpack_codes(codes_g[b * rows:(b + 1) * rows], rows, L.cout, codes_g.shape[1])
            assert np.array_equal(got, f.result()), (L.name, plan.kernel, "codes of image", b)
        del acc[i]
        acc.insert(i, None)
    pool.shutdown()
    return kernels


def test_config3_resnet50_every_layer_full_batch():
    """BJ configs[2]: all 52 LUT convs of ResNet-50 at batch 256."""
    kernels = check_network(3, 256, [0, 85, 170, 255])
    tags = set(kernels.values())
    # the default instances the step relies on were all exercised here
    assert any(t.startswith("f4conv bn=64 win wbres wpair ") for t in tags), tags             # 3x3 64 -> 64: FP4 window pairs
    assert any(t.startswith("f4conv bn=128 win wbres wpair ") for t in tags), tags            # 3x3 128 -> 128: FP4 window pairs
    assert any(" asm " in t for t in tags), tags                                              # short-K 1x1
    assert any(t.startswith("f4conv bn=256") and "direct=1" in t for t in tags), tags         # 1x1 K >= 256: FP4
    assert any(t.startswith("f4conv bn=128") and "direct=1" in t for t in tags), tags         # 1x1 into 128
    assert any(t.startswith("f4conv bn=256") and "direct=0" in t for t in tags), tags         # 3x3 C >= 256: FP4
    assert any(t.startswith("f4conv bn=128") and "direct=0" in t for t in tags), tags         # 3x3 s2 128: FP4
    assert any(t.startswith("f4conv bn=64") and "direct=1" in t for t in tags), tags          # 1x1 256 -> 64: FP4
    assert any(t.startswith("f4conv bn=64 win1x1 ") for t in tags), tags                      # 1x1 64 -> 64: window pairs


def test_config4_vgg16_every_layer_full_batch():
    """BJ configs[3]: all 13 LUT convs of VGG-16 at batch 64 (conv1_1: Cin = 3 padded to 4, im2col)."""
    kernels = check_network(4, 64, [0, 21, 42, 63])
    tags = set(kernels.values())
    assert sum(t.startswith("f4conv bn=128 win wbres wpair ") for t in kernels.values()) == 2, tags   # conv2_1/2_2: 112 wide
    assert any(t.startswith("f4conv bn=64 win wbres wpair ") for t in tags), tags       # conv1_2: FP4 window pairs, 224 wide


def test_config4_conv2d_abi_matches_gemm_path():
    """dg_lut_conv2d (user API, weights expanded per call) == the bench path (prepared weights),
    both already oracle-checked above; here on layers 0 and 3 at batch 8."""
    r = netrun.NetRunner(4, range(8), "cuda", layers=[0, 3])
    r.step()
    ref = [p.out.clone() for p in r.plans]
    for p in r.plans:
        p.out.zero_()
    r.step_conv2d()
    torch.cuda.synchronize()
    for a, p in zip(ref, r.plans):
        assert torch.equal(a, p.out)


def oracle_resnet18_chain():
    """Oracle-side chain of config 2 (parity unpinned by the paper: it prints no network
    outputs; each step is the pinned conv / requant oracle)."""
    L = synth.resnet18_layers()
    rqs = synth.resnet18_requants()
    al = np.array(synth.AL_UNIFORM, np.int64)
    x = netrun.input_codes(2, 0, L[0], [0], "cpu").numpy()
    outs = []
    for c1, c2, ds in synth.resnet18_blocks():
        W = {li: netrun.weight_codes(2, li, L[li], "cpu").numpy() for li in (c1, c2) + ((ds,) if ds is not None else ())}
        r1, _ = rqs[c1]
        a1 = oracle.conv2d_direct(x, W[c1], T_CONV, L[c1].stride, L[c1].pad, 0).reshape(-1, L[c1].cout)
        y1 = oracle.requantize(a1, r1.mult, r1.shift, r1.zp, r1.qmin, r1.qmax,
                               bias=np.full(L[c1].cout, r1.bias, np.int32), bias_axis=0)
        y1 = y1.reshape(1, L[c1].ho, L[c1].ho, L[c1].cout)
        a2 = oracle.conv2d_direct(y1, W[c2], T_CONV, L[c2].stride, L[c2].pad, 0).reshape(-1, L[c2].cout)
        r2, res_mult = rqs[c2]
        if ds is not None:
            res = oracle.conv2d_direct(x, W[ds], T_CONV, L[ds].stride, L[ds].pad, 0).reshape(-1, L[ds].cout)
        else:
            res = (al[x.reshape(-1, L[c2].cout)] * res_mult).astype(np.int32)
        out = oracle.requantize(a2, r2.mult, r2.shift, r2.zp, r2.qmin, r2.qmax, res=res,
                                bias=np.full(L[c2].cout, r2.bias, np.int32), bias_axis=0)
        x = out.reshape(1, L[c2].ho, L[c2].ho, L[c2].cout)
        outs.append(x)
    return outs


def test_config2_resnet18_chain_bit_exact():
    r = netrun.ResNet18Runner("cuda")
    r.step()
    torch.cuda.synchronize()
    ref = oracle_resnet18_chain()
    for bi, ((c1, c2, ds), (y1, out, racc)) in enumerate(zip(r.blocks, r.bufs)):
        L2 = r.layers[c2]
        g = out.cpu().numpy()
        got = oracle.unpack_codes(g, g.shape[0], L2.cout, g.shape[1])
        assert np.array_equal(got, ref[bi].reshape(-1, L2.cout)), f"block {bi}"
    # the codes are spread (the chain did not collapse to a constant)
    hist = np.bincount(ref[-1].ravel(), minlength=4) / ref[-1].size
    assert (hist > 0.02).sum() >= 3, hist


@pytest.mark.parametrize("bmc", [1, 0])
@pytest.mark.parametrize("n", [4096])
def test_config5_square_gemm_freivalds(n, bmc):
    """Config 5 (Q17 learned levels, int16 table, int32 out) at n=4096, with the B stages multicast
    across 2-CTA clusters (bmc = 1) and without (the default): exact Freivalds over the whole C and
    two full rows against the oracle."""
    dg.reset_options()
    dg.set_option("bmc", bmc)
    wl, al = synth.learned_levels(5, 0, synth.T_LEVELS)
    lut = dg.build_lut(wl, al, 16)
    Wc = synth.counter_codes_host(0, n * n, (5, n, synth.T_W), "uniform").reshape(n, n)
    Ac = synth.counter_codes_host(0, n * n, (5, n, synth.T_A), "uniform").reshape(n, n)
    w = dg.pack_weights(torch.from_numpy(Wc).cuda())
    at = dg.pack_codes(torch.from_numpy(Ac).cuda())
    at8 = dg.expand_operand(at, n, al)
    C = dg.lut_gemm_prepared(w, at8, n, n, n, lut)
    tag = dg.last_kernel()
    C2 = dg.lut_gemm(w, at, n, n, n, lut, variant="tc")
    torch.cuda.synchronize()
    dg.reset_options()
    assert f"bmc={bmc}" in tag and "bn=256" in tag, tag
    assert torch.equal(C, C2)
    Cn = C.cpu().numpy()
    T = oracle.build_lut16(wl, al)
    assert oracle.freivalds_rows(Wc, Ac, Cn, T, trials=2) == 0
    rows = [0, n - 1]
    assert np.array_equal(oracle.lut_gemm(Wc[rows], np.ascontiguousarray(Ac.T), T), Cn[rows])
