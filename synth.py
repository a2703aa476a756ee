"""Seeded synthetic inputs and workload shapes for the five BASELINE.json configs.

This module is shared by the oracle side (tests) and the CUDA side (tests,
bench.py, smoke).  It holds NONE of the method's arithmetic: it only draws
codes / level sets from seeded generators and lists layer shapes.  Every draw
comes from ``numpy.random.Generator(PCG64(SeedSequence(MASTER_SEED,
spawn_key=(cfg, layer, tensor_id, image))))`` so any shard regenerates exactly
its own images and any GPU count sees identical data.

Recipe (BASELINE.json configs):
  * weight codes       i.i.d. uniform over {0,1,2,3}
  * activation codes   uniform (configs 1, 5) or ReLU-skewed: P(0)=0.5, else
                       uniform over {1,2,3} (configs 2-4)
  * levels             configs 1-4: wl[c] = c-2, al[c] = c (reading Q2);
                       config 5: learned-style levels (reading Q17)
  * requant            per-layer fixed point, shift 20 (reading Q12)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MASTER_SEED = 230409049

# tensor ids inside a spawn key
T_W, T_A, T_X, T_LEVELS, T_RES = 0, 1, 2, 3, 4

WL_UNIFORM = (-2, -1, 0, 1)   # BJ configs[0]: weight codes {0..3} -> levels {-2,-1,0,1} (Q2)
AL_UNIFORM = (0, 1, 2, 3)     # BJ configs[0]: activation codes {0..3} -> levels {0..3}


def rng(*key: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(MASTER_SEED, spawn_key=tuple(key))))


def uniform_codes(shape, *key: int) -> np.ndarray:
    return rng(*key).integers(0, 4, size=shape, dtype=np.uint8)


def relu_codes(shape, *key: int) -> np.ndarray:
    """P(0)=0.5, the rest uniform over {1,2,3} (BJ configs[1])."""
    g = rng(*key)
    zero = g.random(size=shape) < 0.5
    nz = g.integers(1, 4, size=shape, dtype=np.uint8)
    return np.where(zero, np.uint8(0), nz).astype(np.uint8)


def learned_levels(*key: int):
    """Config 5 (reading Q17): 4 weight levels ~ N(0,1), 4 activation levels ~ |N(0,1)|,
    each set sorted ascending and scaled by 127/max|.|, rounded half away from zero."""
    g = rng(*key)
    w = np.sort(g.standard_normal(4))
    a = np.sort(np.abs(g.standard_normal(4)))

    def scale(v):
        s = 127.0 / np.max(np.abs(v))
        return [int(math.copysign(math.floor(abs(x * s) + 0.5), x)) for x in v]

    return tuple(scale(w)), tuple(scale(a))


# ---------------------------------------------------------------------------
# Requant parameters (reading Q12).  They depend only on the input
# distribution, never on computed outputs.

@dataclass(frozen=True)
class Requant:
    mult: int
    shift: int
    zp: int
    qmin: int
    qmax: int
    bias: int            # same value for every output channel


def level_moments(levels, probs):
    e1 = sum(l * p for l, p in zip(levels, probs))
    e2 = sum(l * l * p for l, p in zip(levels, probs))
    return e1, e2


P_UNIFORM = (0.25, 0.25, 0.25, 0.25)
P_RELU = (0.5, 1 / 6, 1 / 6, 1 / 6)


def requant_for(K: int, a_probs, gain: float, zp: int, shift: int = 20, extra_var: float = 0.0,
                extra_mean: float = 0.0) -> Requant:
    ew, ew2 = level_moments(WL_UNIFORM, P_UNIFORM)
    ea, ea2 = level_moments(AL_UNIFORM, a_probs)
    mu = K * ew * ea + extra_mean
    var = K * (ew2 * ea2 - (ew * ea) ** 2) + extra_var
    sigma = math.sqrt(var)
    return Requant(mult=int(round((1 << shift) * gain / sigma)), shift=shift, zp=zp, qmin=0, qmax=3,
                   bias=-int(round(mu)))


# config 1 values printed in SURVEY §8(c) Q12: mu=-432, sigma=51.96 -> bias 432, mult 20180, zp 1
CFG1 = dict(M=64, N=196, K=576)
CFG1_RQ = requant_for(576, P_UNIFORM, 1.0, zp=1)


# ---------------------------------------------------------------------------
# Layer shapes (standard torchvision architectures, v1.5
# stride placement for ResNet-50, reading Q15).

@dataclass(frozen=True)
class ConvLayer:
    name: str
    cin: int
    cout: int
    k: int
    stride: int
    pad: int
    h: int              # input spatial size (square)
    chain_in: str = ""  # config 2: which tensor feeds it
    role: str = ""      # config 2: "c1" | "c2" | "ds"

    @property
    def ho(self) -> int:
        return (self.h + 2 * self.pad - self.k) // self.stride + 1

    @property
    def K(self) -> int:
        return self.k * self.k * self.cin

    def gemm_mnk(self, batch: int):
        return self.cout, batch * self.ho * self.ho, self.K

    def ops(self, batch: int) -> int:
        M, N, K = self.gemm_mnk(batch)
        return 2 * M * N * K


def resnet18_layers():
    """19 LUT convs of ResNet-18 at 224x224 (layer1..layer4, incl. 3 downsample 1x1)."""
    L = []
    h = 56
    cin = 64
    for stage, cout in enumerate((64, 128, 256, 512)):
        for blk in range(2):
            s = 2 if (blk == 0 and stage > 0) else 1
            name = f"layer{stage + 1}.{blk}"
            L.append(ConvLayer(f"{name}.conv1", cin, cout, 3, s, 1, h, role="c1"))
            ho = (h + 2 - 3) // s + 1
            L.append(ConvLayer(f"{name}.conv2", cout, cout, 3, 1, 1, ho, role="c2"))
            if s != 1 or cin != cout:
                L.append(ConvLayer(f"{name}.downsample", cin, cout, 1, s, 0, h, role="ds"))
            cin, h = cout, ho
    return L


def resnet50_layers():
    """52 LUT convs of ResNet-50 v1.5 at 224x224 (16 bottlenecks x 3 + 4 downsample)."""
    L = []
    h = 56
    cin = 64
    for stage, (width, nblk) in enumerate(((64, 3), (128, 4), (256, 6), (512, 3))):
        cout = width * 4
        for blk in range(nblk):
            s = 2 if (blk == 0 and stage > 0) else 1
            name = f"layer{stage + 1}.{blk}"
            L.append(ConvLayer(f"{name}.conv1", cin, width, 1, 1, 0, h))
            L.append(ConvLayer(f"{name}.conv2", width, width, 3, s, 1, h))
            ho = (h + 2 - 3) // s + 1
            L.append(ConvLayer(f"{name}.conv3", width, cout, 1, 1, 0, ho))
            if blk == 0:
                L.append(ConvLayer(f"{name}.downsample", cin, cout, 1, s, 0, h))
            cin, h = cout, ho
    return L


def vgg16_layers():
    """13 3x3 convs of VGG-16 at 224x224; conv1_1 has Cin=3 (padded to 4 channels)."""
    spec = [(3, 64, 224), (64, 64, 224), (64, 128, 112), (128, 128, 112), (128, 256, 56),
            (256, 256, 56), (256, 256, 56), (256, 512, 28), (512, 512, 28), (512, 512, 28),
            (512, 512, 14), (512, 512, 14), (512, 512, 14)]
    return [ConvLayer(f"conv{i}", ci, co, 3, 1, 1, h) for i, (ci, co, h) in enumerate(spec)]


CONFIG_LAYERS = {2: resnet18_layers, 3: resnet50_layers, 4: vgg16_layers}
CONFIG_BATCH = {2: 1, 3: 256, 4: 64}
CONFIG_NAMES = {1: "gemm_64x196x576", 2: "resnet18_b1", 3: "resnet50_b256", 4: "vgg16_b64",
                5: "square_gemm"}


def conv_requant(layer: ConvLayer) -> Requant:
    """Per-layer requant for configs 2-4 (ReLU-skewed input codes, gain 1.5, zp 0; Q12)."""
    return requant_for(layer.K, P_RELU, 1.5, zp=0)


def conv_input_codes(cfg: int, li: int, layer: ConvLayer, images) -> np.ndarray:
    """Per-layer independent NHWC input codes [len(images)][h][h][cin] (reading Q16),
    drawn per image so that a batch shard regenerates only its own images."""
    out = np.empty((len(images), layer.h, layer.h, layer.cin), np.uint8)
    for i, b in enumerate(images):
        out[i] = relu_codes((layer.h, layer.h, layer.cin), cfg, li, T_X, int(b))
    return out


def conv_weight_codes(cfg: int, li: int, layer: ConvLayer) -> np.ndarray:
    """[cout][k][k][cin] codes, uniform."""
    return uniform_codes((layer.cout, layer.k, layer.k, layer.cin), cfg, li, T_W)


# ---------------------------------------------------------------------------
# Counter-based generator for the large workloads (configs 2-5).  Implemented once in
# torch integer ops, so the SAME code produces identical codes on CPU (oracle side,
# for sampled images) and on the GPU (bench inputs): code[i] = f(hash(key, i)).
# splitmix64 finaliser with logical shifts emulated on int64.

_M64 = (1 << 64) - 1


def _s64(v: int) -> int:
    v &= _M64
    return v - (1 << 64) if v >= (1 << 63) else v


_GOLD = _s64(0x9E3779B97F4A7C15)
_MIX1 = _s64(0xBF58476D1CE4E5B9)
_MIX2 = _s64(0x94D049BB133111EB)


def _key64(key) -> int:
    h = MASTER_SEED
    for k in key:
        h = (h * 0x100000001B3 + int(k) + 0x9E37) & _M64
        h ^= h >> 29
    return _s64(h)


def _lsr(t, s: int):
    import torch
    return (t >> s) & ((1 << (64 - s)) - 1)


def counter_hash(start: int, count: int, key, device="cpu"):
    """64-bit hashes of element indices [start, start+count) under `key` (int64 tensor)."""
    import torch
    idx = torch.arange(start, start + count, dtype=torch.int64, device=device)
    z = idx * _GOLD + _key64(key)
    z = (z ^ _lsr(z, 30)) * _MIX1
    z = (z ^ _lsr(z, 27)) * _MIX2
    return z ^ _lsr(z, 31)


def counter_codes(start: int, count: int, key, dist: str = "uniform", device="cpu"):
    """uint8 codes for flat element indices [start, start+count).
    dist 'uniform': U{0..3};  'relu': P(0)=1/2, else U{1,2,3} (up to 2^-31 bias)."""
    import torch
    z = counter_hash(start, count, key, device)
    r = z & 0xFFFFFFFF
    if dist == "uniform":
        return (r & 3).to(torch.uint8)
    half = 1 << 31
    nz = 1 + (((r - half).clamp(min=0) * 3) >> 31)
    return torch.where(r < half, torch.zeros_like(r), nz).to(torch.uint8)


_SG = None


def _sg_lib():
    """synth_gen.c (the same counter generator in C + OpenMP), compiled on first use."""
    global _SG
    if _SG is None:
        import ctypes
        import os
        import subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        src, lib = os.path.join(here, "synth_gen.c"), os.path.join(here, "synth_gen.so")
        if not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(src):
            tmp = lib + f".{os.getpid()}.tmp"
            subprocess.check_call(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", src, "-o", tmp])
            os.replace(tmp, lib)
        L = ctypes.CDLL(lib)
        L.sg_counter_codes.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p]
        _SG = L
    return _SG


def counter_codes_host(start: int, count: int, key, dist: str = "uniform") -> np.ndarray:
    """counter_codes on the host as a numpy uint8 array (synth_gen.c; identical values)."""
    out = np.empty(count, np.uint8)
    _sg_lib().sg_counter_codes(start, count, _key64(key) & _M64, 0 if dist == "uniform" else 1,
                               out.ctypes.data)
    return out


def counter_codes_chunked(start: int, count: int, key, dist: str = "uniform", device="cpu", chunk: int = 1 << 24):
    """counter_codes for large counts without int64 temporaries of the full size."""
    import torch
    out = torch.empty(count, dtype=torch.uint8, device=device)
    for s in range(0, count, chunk):
        e = min(count, s + chunk)
        out[s:e] = counter_codes(start + s, e - s, key, dist, device)
    return out


# ---------------------------------------------------------------------------
# Config 2 (ResNet-18 at batch 1, chained, residual adds in int32 before requant; Q13)

def resnet18_blocks():
    """[(conv1, conv2, downsample_or_None)] of the 8 basic blocks (indices into resnet18_layers())."""
    L = resnet18_layers()
    blocks, i = [], 0
    while i < len(L):
        c1, c2 = i, i + 1
        ds = i + 2 if i + 2 < len(L) and L[i + 2].role == "ds" else None
        blocks.append((c1, c2, ds))
        i += 3 if ds is not None else 2
    return blocks


def resnet18_requants():
    """Per-layer requant (Q12) and per-block residual scale (Q13).  Uses the calibration in
    synth_data/resnet18_requant.json (written by tools/calibrate_resnet18.py from the CPU oracle
    chain only) when present; otherwise analytic values from the input distribution."""
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "synth_data", "resnet18_requant.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)["layers"]
        return {int(k): ((None if v["mult"] == 0 else Requant(v["mult"], v["shift"], v["zp"], 0, 3, v["bias"])),
                         v["res_mult"]) for k, v in d.items()}
    L = resnet18_layers()
    out = {}
    ea, ea2 = level_moments(AL_UNIFORM, P_RELU)
    var_a = ea2 - ea * ea
    ew, ew2 = level_moments(WL_UNIFORM, P_UNIFORM)
    for c1, c2, ds in resnet18_blocks():
        out[c1] = (conv_requant(L[c1]), 0)
        K2 = L[c2].K
        sig2 = math.sqrt(K2 * (ew2 * ea2 - (ew * ea) ** 2))
        if ds is None:
            res_mult = max(1, int(round(sig2 / math.sqrt(var_a))))
            extra_mean, extra_var = res_mult * ea, res_mult * res_mult * var_a
        else:
            res_mult = 0
            Kd = L[ds].K
            extra_mean, extra_var = Kd * ew * ea, Kd * (ew2 * ea2 - (ew * ea) ** 2)
            out[ds] = (None, 0)
        out[c2] = (requant_for(K2, P_RELU, 1.5, zp=0, extra_var=extra_var, extra_mean=extra_mean), res_mult)
    return out
