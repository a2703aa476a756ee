"""Launch-overlap stress (compute-sanitizer is not available on this GPU pool, profiles/
r02_compute_sanitizer_closed.txt): a CHAIN of convolutions where every layer reads the previous
layer's packed output, one layer per kernel instance of the auto dispatch (window pair / tile
modes, short-K shared-memory A, 128x256 long-K, implicit stride-2 gather, direct 1x1, split-K +
reduce), captured in one CUDA graph with programmatic dependent launch and the early_weights
contract (the bench's regime), replayed many times; after every replay each layer's output must
equal the oracle's chain bit for bit.  A consumer reading its producer's output before the
producer finished (a missing griddepcontrol.wait) shows up here as a mismatch."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2304_09049_b200 import dg  # noqa: E402

WL, AL = [-2, -1, 0, 1], [0, 1, 2, 3]
# (Cout, k, stride, expected instance tag fragment); input 24 x 40 x 40 x 64 codes
CHAIN = [
    (64, 3, 1, " win "),            # C = 64 window (pair mode at this size)
    (256, 1, 1, " asm "),           # short-K 1x1, A in shared memory
    (128, 1, 1, "bn=128"),          # 256 -> 128 direct, short K
    (128, 3, 1, "kst=128 win"),     # C = 128 window tile mode
    (128, 3, 2, "implicit=1"),      # stride-2 implicit gather
    (512, 1, 1, " asm "),
    (256, 1, 1, "bn=128 epi=4"),    # K = 512 long-K (few tiles: 128-wide)
    (256, 3, 1, "implicit=1"),      # 3x3 C = 256 implicit gather
    (256, 3, 2, "skinst"),          # few output tiles: split-K + reduce kernel
]


def test_conv_chain_graph_replays_bit_exact():
    g = np.random.default_rng(2024)
    B, H, C = 24, 40, 64
    T = oracle.build_lut16(WL, AL)
    x = g.integers(0, 4, (B, H, H, C), dtype=np.uint8)
    lut = dg.build_lut(WL, AL, 8)
    dev = "cuda"
    cur = dg.pack_codes(torch.from_numpy(x.reshape(-1, C)).to(dev))[:, : C // 4].contiguous()
    layers, exp = [], []
    xo, h, c = x, H, C
    for li, (cout, k, s, frag) in enumerate(CHAIN):
        w = g.integers(0, 4, (cout, k, k, c), dtype=np.uint8)
        pad = k // 2
        acc = oracle.conv2d_direct(xo, w, T, s, pad, 0)
        ho = acc.shape[1]
        a2 = acc.reshape(-1, cout).astype(np.float64)
        bias = (-np.round(a2.mean(axis=0))).astype(np.int32)          # per channel (folded-BN style)
        mult = int(round((1 << 20) / max(1.0, float((a2 + bias).std()))))
        codes = oracle.requantize(acc.reshape(-1, cout), mult, 20, 1, 0, 3, bias=bias, bias_axis=0)
        wp = dg.pack_weights(torch.from_numpy(w.reshape(cout, -1)).to(dev))
        w8 = dg.expand_operand(wp, k * k * c, WL)
        p = dg.conv_params(B, h, h, c, cout, k, k, s, pad, 0, ldw=wp.shape[1])
        out = torch.empty((B * ho * ho, cout // 4), dtype=torch.uint8, device=dev)
        rq = dg.Requant(mult, 20, 1, 0, 3, bias=torch.from_numpy(bias).to(dev), bias_axis=0)
        ws = torch.zeros(max(16, dg.conv_workspace_size(p)), dtype=torch.uint8, device=dev)
        layers.append((cur, w8, p, rq, out, ws, frag))
        exp.append(codes)
        cur, xo, h, c = out, codes.reshape(B, ho, ho, cout), ho, cout
    torch.cuda.synchronize()

    def step():
        tags = []
        for (xin, w8, p, rq, out, ws, frag) in layers:
            dg.lut_conv2d_prepared(xin, w8, lut, p, rq=rq, out=out, ws=ws)
            tags.append(dg.last_kernel())
        return tags

    with dg.options(early_weights=1):
        tags = step()
        for t, (*_, frag) in zip(tags, layers):
            assert frag in t, (frag, t)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
    for rep in range(25):
        for (*_, out, ws, frag) in layers:
            out.fill_(0x5A)                  # poison: a premature read would see this
        graph.replay()
        torch.cuda.synchronize()
        for li, ((*_, out, ws, frag), e) in enumerate(zip(layers, exp)):
            got = oracle.unpack_codes(out.cpu().numpy(), e.shape[0], e.shape[1], out.shape[1])
            assert np.array_equal(got, e), (rep, li, frag)
    # the chain's codes stay spread (it did not collapse to a constant)
    assert (np.bincount(exp[-1].ravel(), minlength=4) > exp[-1].size // 50).sum() >= 3


# the same regime on the FP4 conv kernel (dg_lut_conv2d_f4_prepared): shifted-window pairs (64- and
# 128-wide, resident weights; the 1x1 64 -> 64 window pairs), direct 1x1 tiles of every width, the im2col-mode strided 1x1, the
# gathered stride-2 3x3; input 24 x 40 x 40 x 64 codes
F4_CHAIN = [
    (64, 3, 1, "bn=64 win wbres wpair"),
    (64, 1, 1, "bn=64 win1x1 wbres wpair"),
    (128, 3, 1, "bn=128 win wbres wpair"),
    (128, 3, 1, "bn=128 win wbres wpair"),
    (256, 1, 2, "direct=1 i2c"),
    (64, 1, 1, "bn=64 ta nacc=4"),
    (256, 1, 1, "bn=256 ta nacc=1"),
    (256, 3, 2, "direct=0"),
    (512, 1, 1, "bn=256 ta nacc=1"),
]


def test_f4_conv_chain_graph_replays_bit_exact():
    g = np.random.default_rng(2025)
    B, H, C = 24, 40, 64
    T = oracle.build_lut16(WL, AL)
    x = g.integers(0, 4, (B, H, H, C), dtype=np.uint8)
    lut = dg.build_lut(WL, AL, 8)
    dev = "cuda"
    cur = dg.pack_codes(torch.from_numpy(x.reshape(-1, C)).to(dev))[:, : C // 4].contiguous()
    layers, exp = [], []
    xo, h, c = x, H, C
    for cout, k, s, frag in F4_CHAIN:
        w = g.integers(0, 4, (cout, k, k, c), dtype=np.uint8)
        pad = k // 2
        acc = oracle.conv2d_direct(xo, w, T, s, pad, 0)
        ho = acc.shape[1]
        a2 = acc.reshape(-1, cout).astype(np.float64)
        bias = (-np.round(a2.mean(axis=0))).astype(np.int32)
        wp = dg.pack_weights(torch.from_numpy(w.reshape(cout, -1)).to(dev))
        w4 = dg.expand_operand_f4(wp, k * k * c, WL)
        p = dg.conv_params(B, h, h, c, cout, k, k, s, pad, 0, ldw=wp.shape[1])
        out = torch.empty((B * ho * ho, cout // 4), dtype=torch.uint8, device=dev)
        bias_d = torch.from_numpy(bias).to(dev)
        # the FP4 kernel takes only requant maps with a 16-bit form (host-verified): the first
        # multiplier from the calibrated one up that has one
        mult = int(round((1 << 20) / max(1.0, float((a2 + bias).std()))))
        for _ in range(64):
            rq = dg.Requant(mult, 20, 1, 0, 3, bias=bias_d, bias_axis=0)
            try:
                dg.lut_conv2d_f4_prepared(cur, w4, lut, p, rq=rq, out=out)
                break
            except dg.DGError:
                mult += 7
        else:
            raise AssertionError(("no 16-bit requant form near", frag))
        codes = oracle.requantize(acc.reshape(-1, cout), mult, 20, 1, 0, 3, bias=bias, bias_axis=0)
        layers.append((cur, w4, p, rq, out, frag))
        exp.append(codes)
        cur, xo, h, c = out, codes.reshape(B, ho, ho, cout), ho, cout
    torch.cuda.synchronize()

    def step():
        tags = []
        for li, (xin, w4, p, rq, out, frag) in enumerate(layers):
            dg.lut_conv2d_f4_prepared(xin, w4, lut, p, rq=rq, out=out)
            tags.append(dg.last_kernel())
        return tags

    dg.reset_options()
    with dg.options(early_weights=1):
        tags = step()
        for t, (*_, frag) in zip(tags, layers):
            assert frag in t, (frag, t)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
    for rep in range(25):
        for (*_, out, frag) in layers:
            out.fill_(0x5A)                  # poison: a premature read would see this
        graph.replay()
        torch.cuda.synchronize()
        for li, ((*_, out, frag), e) in enumerate(zip(layers, exp)):
            got = oracle.unpack_codes(out.cpu().numpy(), e.shape[0], e.shape[1], out.shape[1])
            assert np.array_equal(got, e), (rep, li, frag)
    assert (np.bincount(exp[-1].ravel(), minlength=4) > exp[-1].size // 50).sum() >= 3
