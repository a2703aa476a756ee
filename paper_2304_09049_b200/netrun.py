"""Layer-by-layer runner for the conv workloads (BASELINE configs 3 and 4) on one GPU.

Builds every layer's packed weights, packed NHWC input codes, requant parameters and
output buffers in HBM, then runs one *step* = every LUT conv of the network over the
local batch shard (reading Q16: per-layer independent inputs).  Each layer is
im2col (S3, when the layer is not a plain 1x1/stride-1 conv) -> LUT GEMM with the
fused requant epilogue (S5-S7), issued through the C ABI (dg_im2col, dg_lut_gemm), or
through dg_lut_conv2d for the user-level path.

Inputs are drawn with synth.counter_codes (the same counter-based generator the oracle
side uses), indexed by global image id, so any shard of images is reproducible.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import dg


def _synth():
    import synth  # seeded input generators (no method arithmetic), repo root
    return synth


@dataclass
class LayerPlan:
    name: str
    layer: object
    params: object
    lut: object            # product table, index (w<<2)|a (dg_lut_conv2d orientation)
    lut_t: object          # transposed table, index (a<<2)|w (dg_lut_gemm with P = pixels)
    rq: object
    w: torch.Tensor        # packed weights [Cout][ldw]
    w8: torch.Tensor | None  # int8 level expansion of w (offline, tc path), dg_expand_operand
    x: torch.Tensor        # packed NHWC input [B*H*W][Cp/4]
    out: torch.Tensor      # packed NHWC output codes [B*Ho*Wo][Cout/4]
    rows: int              # B*Ho*Wo  (GEMM rows on the P side)
    K: int                 # computed reduction length (padded channels)
    direct: bool           # 1x1 / stride 1 / unpadded: the input is its own im2col matrix
    ops: int               # algorithmic 2*M*N*K with the unpadded K
    kernel: str = ""       # dg_last_kernel() tag of the GEMM instance the layer ran (last step)
    w4: torch.Tensor | None = None   # e2m1 expansion of w (FP4 conv kernel), dg_expand_operand_f4

    @property
    def cols_ld(self) -> int:
        return dg.packed_ld(self.K)

    @property
    def implicit(self) -> bool:
        """tc path gathers im2col rows on chip (dg_lut_conv2d_prepared): C/4 a power of two >= 16."""
        cb = self.params.C // 4
        return (not self.direct) and cb >= 16 and (cb & (cb - 1)) == 0 and self.layer.k * self.layer.k <= 64


def f4_default(layer, Cp: int) -> bool:
    """Layers the block-scaled FP4 conv kernel (dg_lut_conv2d_f4_prepared, A operand in tensor
    memory; 256-wide tiles where 256 divides Cout, 64-wide for Cout = 64, else 128; 8 epilogue
    warps) takes by default, from per-layer measurements against the int8 kernels (DESIGN.md
    §6.4): 1x1 convs with K >= 256 (stride 1 or 2, Cout = 64 or >= 128) or into 64 channels, the
    gathered 3x3 convs over >= 256 channels, the 3x3 convs over 128 channels that are strided or
    produce a multiple of 256 channels, and the 3x3 s1 convs from 64 / 128 into 64 / 128 channels
    (shifted window with resident weights, one window per two 128-row blocks).  The short-K wide 1x1
    layers (K <= 128 into >= 128 channels) stay on int8."""
    K = layer.k * layer.k * Cp
    if layer.cout % 4 or not (layer.cout >= 128 or layer.cout == 64):
        return False
    if layer.k == 1 and layer.pad == 0:
        return K >= 256 or layer.cout == 64
    if layer.k == 3 and layer.stride == 1 and layer.pad == 1 and Cp in (64, 128) and layer.cout in (64, 128):
        return True   # shifted window, resident weights, window pairs
    return layer.cout >= 128 and layer.k == 3 and (Cp >= 256 or (Cp >= 128 and (layer.cout % 256 == 0 or layer.stride == 2)))


def input_codes(cfg: int, li: int, layer, images, device):
    """NHWC codes [len(images)][h][h][cin] of layer li for global image ids `images`
    (contiguous ids), drawn with the counter generator."""
    s = _synth()
    per = layer.h * layer.h * layer.cin
    b0 = int(images[0])
    n = len(images)
    c = s.counter_codes(b0 * per, n * per, (cfg, li, s.T_X), "relu", device)
    return c.view(n, layer.h, layer.h, layer.cin)


def weight_codes(cfg: int, li: int, layer, device):
    s = _synth()
    n = layer.cout * layer.k * layer.k * layer.cin
    return s.counter_codes(0, n, (cfg, li, s.T_W), "uniform", device).view(layer.cout, layer.k, layer.k, layer.cin)


def pack_nhwc(codes: torch.Tensor) -> torch.Tensor:
    """[B][H][W][C] codes -> packed NHWC [B*H*W][Cp/4] (Cp = roundup(C,4); pad channels code 0)."""
    B, H, W, C = codes.shape
    Cp = (C + 3) // 4 * 4
    flat = codes.reshape(-1, C)
    if Cp != C:
        z = torch.zeros((flat.shape[0], Cp), dtype=torch.uint8, device=codes.device)
        z[:, :C] = flat
        flat = z
    packed = dg.pack_codes(flat.contiguous())
    if packed.shape[1] != Cp // 4:
        packed = packed[:, :Cp // 4].contiguous()
    return packed


def pack_conv_weights(w: torch.Tensor, wpad_code: int = 2) -> torch.Tensor:
    """[Cout][k][k][C] -> packed [Cout][ldw] over K = k*k*Cp; pad channels get a zero-level code."""
    Cout, kh, kw, C = w.shape
    Cp = (C + 3) // 4 * 4
    if Cp != C:
        z = torch.full((Cout, kh, kw, Cp), wpad_code, dtype=torch.uint8, device=w.device)
        z[..., :C] = w
        w = z
    return dg.pack_weights(w.reshape(Cout, -1).contiguous())


class NetRunner:
    def __init__(self, cfg: int, images, device="cuda", variant="auto", layers=None, f4=None):
        """f4: layer ids to run on the block-scaled FP4 conv kernel (dg_lut_conv2d_f4_prepared), or
        None for the default selection f4_default(layer)."""
        s = _synth()
        self.cfg = cfg
        self.images = list(images)
        self.B = len(self.images)
        self.device = device
        self.variant = variant
        all_layers = s.CONFIG_LAYERS[cfg]()
        self.layer_ids = list(range(len(all_layers))) if layers is None else list(layers)
        wl, al = s.WL_UNIFORM, s.AL_UNIFORM
        lut = dg.build_lut(wl, al, 8)
        lut_t = dg.build_lut(al, wl, 8)
        self.plans: list[LayerPlan] = []
        ws_need = 0
        for li in self.layer_ids:
            L = all_layers[li]
            Cp = (L.cin + 3) // 4 * 4
            K = L.k * L.k * Cp
            wq = pack_conv_weights(weight_codes(cfg, li, L, device))
            xq = pack_nhwc(input_codes(cfg, li, L, self.images, device))
            params = dg.conv_params(self.B, L.h, L.h, Cp, L.cout, L.k, L.k, L.stride, L.pad, 0, ldw=wq.shape[1])
            rows = self.B * L.ho * L.ho
            r = s.conv_requant(L)
            bias = torch.full((L.cout,), r.bias, dtype=torch.int32, device=device)
            rq = dg.Requant(r.mult, r.shift, r.zp, r.qmin, r.qmax, bias=bias, bias_axis=0)
            out = torch.empty((rows, L.cout // 4), dtype=torch.uint8, device=device)
            direct = L.k == 1 and L.stride == 1 and L.pad == 0 and (Cp // 4) % 16 == 0
            w8 = dg.expand_operand(wq, K, wl) if variant in ("auto", "tc") else None
            plan = LayerPlan(L.name, L, params, lut, lut_t, rq, wq, w8, xq, out, rows, K, direct,
                             2 * L.cout * rows * L.k * L.k * L.cin)
            use_f4 = (li in f4) if f4 is not None else (variant == "auto" and f4_default(L, Cp))
            if use_f4:
                plan.w4 = dg.expand_operand_f4(wq, K, wl)
            ws_need = max(ws_need, dg.conv_workspace_size(params), (0 if direct else rows * plan.cols_ld),
                          dg.gemm_workspace_size(rows, L.cout, K))
            self.plans.append(plan)
        self.ws = torch.zeros(max(ws_need, 16), dtype=torch.uint8, device=device)
        self.ws_gemm = self.ws
        self.total_ops = sum(p.ops for p in self.plans)

    # -- the step, split into C-ABI calls so the GEMM launches can be bracketed by events
    def step(self, gemm_events=None, stream=None, int32_out=None):
        """One step: every layer, requantised codes into plan.out, or (int32_out = one int32
        [rows][Cout] buffer per layer) the raw accumulators of the same kernel instances."""
        n = 0
        for i, p in enumerate(self.plans):
            L = p.layer
            if p.w4 is not None:   # block-scaled FP4 conv kernel
                if gemm_events is not None:
                    gemm_events[i][0].record()
                dg.lut_conv2d_f4_prepared(p.x, p.w4, p.lut, p.params, rq=None if int32_out else p.rq,
                                          out=int32_out[i] if int32_out else p.out, stream=stream)
                p.kernel = dg.last_kernel()
                if gemm_events is not None:
                    gemm_events[i][1].record()
                n += 1
                continue
            if p.w8 is not None and (p.direct or p.implicit):
                # tensor-core path without an im2col matrix (direct 1x1 or implicit GEMM)
                if gemm_events is not None:
                    gemm_events[i][0].record()
                dg.lut_conv2d_prepared(p.x, p.w8, p.lut, p.params, rq=None if int32_out else p.rq,
                                       out=int32_out[i] if int32_out else p.out, ws=self.ws, stream=stream)
                p.kernel = dg.last_kernel()
                if gemm_events is not None:
                    gemm_events[i][1].record()
                n += 1
                continue
            if p.direct:
                P = p.x
            else:
                ld = p.cols_ld
                P = self.ws[: p.rows * ld].view(p.rows, ld)
                if p.w8 is None:   # packed-weights GEMM needs its own workspace after the columns
                    off = (p.rows * ld + 127) // 128 * 128
                    self.ws_gemm = self.ws[off:]
                dg.im2col(p.x, self.B, L.h, L.h, p.params.C, L.k, L.k, L.stride, L.pad, 0, out=P, stream=stream)
                n += 1
            if gemm_events is not None:
                gemm_events[i][0].record()
            if p.w8 is not None:   # tensor-core path with the offline-expanded weights
                dg.lut_gemm_prepared(P, p.w8, p.rows, L.cout, p.K, p.lut_t, rq=None if int32_out else p.rq,
                                     out=int32_out[i] if int32_out else p.out, stream=stream)
                p.kernel = dg.last_kernel()
            else:
                dg.lut_gemm(P, p.w, p.rows, L.cout, p.K, p.lut_t, rq=p.rq, variant=self.variant, out=p.out,
                            ws=self.ws_gemm, stream=stream)
            if gemm_events is not None:
                gemm_events[i][1].record()
            n += 1
        return n  # kernel launches issued

    # -- the user-level path: one dg_lut_conv2d per layer
    def step_conv2d(self, stream=None):
        for i in range(len(self.plans)):
            self.conv2d_layer(i, stream)

    def conv2d_layer(self, i: int, stream=None):
        """One layer through the public dg_lut_conv2d call (weights expanded inside the call)."""
        p = self.plans[i]
        dg.lut_conv2d(p.x, p.w, p.lut, p.params, rq=p.rq, variant=self.variant, out=p.out, ws=self.ws, stream=stream)

    def int32_buffers(self):
        return [torch.empty((p.rows, p.layer.cout), dtype=torch.int32, device=self.device) for p in self.plans]

    def input_bytes(self) -> int:
        return sum(p.x.numel() for p in self.plans)

    def output_bytes(self) -> int:
        return sum(p.out.numel() for p in self.plans)

    def weight_bytes(self) -> int:
        return sum(p.w.numel() for p in self.plans)


class ResNet18Runner:
    """BASELINE config 2: the 19 LUT convs of ResNet-18 at batch 1, CHAINED: each basic block is
    conv1 (fused requant) -> conv2 (+ residual in int32, fused requant); the residual is the
    block input's levels x res_mult (identity, over packed codes) or the int32 accumulator of
    the 1x1 stride-2 downsample conv (reading Q13).  All through dg_lut_conv2d."""

    def __init__(self, device="cuda", variant="auto", batch: int = 1):
        s = _synth()
        self.cfg = 2
        self.B = batch
        self.variant = variant
        self.layers = s.resnet18_layers()
        self.blocks = s.resnet18_blocks()
        rqs = s.resnet18_requants()
        wl, al = s.WL_UNIFORM, s.AL_UNIFORM
        self.lut = dg.build_lut(wl, al, 8)
        self.w = {}
        self.params = {}
        self.rq = {}
        self.res_mult = {}
        self.bias = {}
        ws_need = 0
        self.w8 = {}
        self.prepared = variant in ("auto", "tc")
        for li, L in enumerate(self.layers):
            self.w[li] = pack_conv_weights(weight_codes(2, li, L, device))
            p = dg.conv_params(batch, L.h, L.h, L.cin, L.cout, L.k, L.k, L.stride, L.pad, 0, ldw=self.w[li].shape[1])
            if self.prepared:   # offline int8 expansion of the weights (tensor-core path)
                self.w8[li] = dg.expand_operand(self.w[li], L.K, wl)
            self.params[li] = p
            ws_need = max(ws_need, dg.conv_workspace_size(p))
            r, rm = rqs[li]
            self.rq[li] = r
            self.res_mult[li] = rm
            if r is not None:
                self.bias[li] = torch.full((L.cout,), r.bias, dtype=torch.int32, device=device)
        self.ws = torch.zeros(ws_need, dtype=torch.uint8, device=device)
        L0 = self.layers[0]
        self.x0 = pack_nhwc(input_codes(2, 0, L0, list(range(batch)), device))   # stands in for the stem output (Q14)
        self.bufs = []
        for c1, c2, ds in self.blocks:
            L1, L2 = self.layers[c1], self.layers[c2]
            y1 = torch.empty((batch * L1.ho * L1.ho, L1.cout // 4), dtype=torch.uint8, device=device)
            out = torch.empty((batch * L2.ho * L2.ho, L2.cout // 4), dtype=torch.uint8, device=device)
            racc = None
            if ds is not None:
                Ld = self.layers[ds]
                racc = torch.empty((batch * Ld.ho * Ld.ho, Ld.cout), dtype=torch.int32, device=device)
            self.bufs.append((y1, out, racc))
        self.total_ops = sum(2 * L.cout * batch * L.ho * L.ho * L.K for L in self.layers)

    def _rq(self, li, **kw):
        r = self.rq[li]
        return dg.Requant(r.mult, r.shift, r.zp, r.qmin, r.qmax, bias=self.bias[li], bias_axis=0, **kw)

    def _conv(self, x, li, rq, out, stream):
        if self.prepared:
            dg.lut_conv2d_prepared(x, self.w8[li], self.lut, self.params[li], rq=rq, out=out, ws=self.ws, stream=stream)
        else:
            dg.lut_conv2d(x, self.w[li], self.lut, self.params[li], rq=rq, variant=self.variant, out=out, ws=self.ws,
                          stream=stream)

    def step(self, stream=None):
        x = self.x0
        for (c1, c2, ds), (y1, out, racc) in zip(self.blocks, self.bufs):
            self._conv(x, c1, self._rq(c1), y1, stream)
            if ds is not None:
                self._conv(x, ds, None, racc, stream)
                rq2 = self._rq(c2, res=racc)
            else:
                rq2 = self._rq(c2, res_codes=x, res_mult=self.res_mult[c2], res_levels=_synth().AL_UNIFORM)
            self._conv(y1, c2, rq2, out, stream)
            x = out
        return x

    def launches(self) -> int:
        if self.prepared:      # one kernel per conv (direct / implicit GEMM; all C/4 are powers of two)
            return len(self.layers)
        n = 0
        for li, L in enumerate(self.layers):
            direct = L.k == 1 and L.stride == 1 and L.pad == 0 and (L.cin // 4) % 16 == 0
            n += 2 if direct else 3    # (im2col) + weight expansion + GEMM
        return n
