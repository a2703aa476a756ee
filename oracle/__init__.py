"""Plain CPU oracle for the DeepGEMM (arXiv 2304.09049) 2-bit LUT GEMM/conv path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may import
this package.  The product path (``paper_2304_09049_b200``) never imports it,
and this package never imports the product path: the two share no code.

The arithmetic lives in ``oracle.c`` (plain nested loops, one function per
definition, each citing the PAPER.md passage it follows); this module only
marshals numpy arrays into it.  ``build()`` compiles ``liboracle.so`` with gcc.

Parity status per function (DESIGN.md §4 lists the pins):
  unpack_codes       pinned (hand examples, roundtrip)
  build_lut16        pinned (S:222 values, Table 2 size)
  lut_gemm           pinned (fp64 BLAS closed form, brute force, invariants)
  conv2d_direct      pinned (1x1 == GEMM, border counts, fp64 im2col matmul)
  requantize         pinned (exact Fraction arithmetic over all ties)
  quantize           pinned (Eq. 1 worked examples S:57-59)
  freivalds_rows     pinned (accepts the true C, rejects single-element faults)
  lut_gemm_f64       pinned (fp64 BLAS closed form for float product tables, integer-valued
                     tables equal lut_gemm exactly, brute force via pair counts, linearity)
  conv_freivalds     pinned (accepts or_conv2d_direct's output incl. padding / stride / pad
                     codes, rejects every single-element fault and swapped channels / pixels,
                     equals freivalds_rows on 1x1 convs)
  resnet18_chain     parity unpinned by the paper (it prints no network outputs);
                     pinned only through its per-layer parts above.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain gcc -O2, single thread)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", _SRC, "-o", _LIB, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        i32 = ctypes.c_int32
        lib.or_unpack_codes.argtypes = [P, i64, i64, i64, P]
        lib.or_build_lut16.argtypes = [P, P, P]
        lib.or_lut_gemm.argtypes = [P, P, i64, i64, i64, P, P]
        lib.or_lut_gemm_bits.argtypes = [P, P, i64, i64, i64, i32, P, P]
        lib.or_conv2d_direct_bits.argtypes = [P, P] + [i32] * 9 + [ctypes.c_uint8, i32, P, P]
        lib.or_lut_gemm.restype = ctypes.c_int
        lib.or_conv2d_direct.argtypes = [P, P] + [i32] * 9 + [ctypes.c_uint8, P, P]
        lib.or_conv2d_direct.restype = ctypes.c_int
        lib.or_requantize.argtypes = [P, P, i64, i64, i64, P, i32, i32, i32, i32, i32, i32, P]
        lib.or_quantize.argtypes = [P, i64, ctypes.c_float, ctypes.c_float, i32, i32, P]
        lib.or_freivalds_rows.argtypes = [P, P, P, i64, i64, i64, i64, P, P, P]
        lib.or_freivalds_rows.restype = i64
        lib.or_lut_gemm_f64.argtypes = [P, P, i64, i64, i64, P, P]
        lib.or_conv_freivalds.argtypes = [P, P] + [i32] * 9 + [ctypes.c_uint8, P, P, i64, P, P]
        lib.or_conv_freivalds.restype = i64
        _lib = lib
    return _lib


def _c(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, a.ctypes.data_as(ctypes.c_void_p)


def unpack_codes(packed: np.ndarray, rows: int, K: int, ld: int) -> np.ndarray:
    """Read the documented packed format (code k in byte k>>2, bits 2(k&3))."""
    lib = _load()
    p, pp = _c(packed, np.uint8)
    assert p.size >= rows * ld
    out = np.empty((rows, K), np.uint8)
    lib.or_unpack_codes(pp, rows, K, ld, out.ctypes.data_as(ctypes.c_void_p))
    return out


def build_lut16(wl, al) -> np.ndarray:
    """T[(i<<2)|j] = wl[i]*al[j]."""
    lib = _load()
    w, wp = _c(wl, np.int32)
    a, ap = _c(al, np.int32)
    assert w.size == 4 and a.size == 4
    T = np.empty(16, np.int32)
    lib.or_build_lut16(wp, ap, T.ctypes.data_as(ctypes.c_void_p))
    return T


def lut_gemm(W: np.ndarray, A: np.ndarray, T) -> np.ndarray:
    """C[m][n] = sum_k T[(W[m][k]<<2)|A[k][n]] (Alg. 1).  W [M][K], A [K][N] codes."""
    lib = _load()
    W, Wp = _c(W, np.uint8)
    A, Ap = _c(A, np.uint8)
    T, Tp = _c(T, np.int32)
    M, K = W.shape
    K2, N = A.shape
    assert K == K2 and T.size == 16
    C = np.empty((M, N), np.int32)
    rc = lib.or_lut_gemm(Wp, Ap, M, N, K, Tp, C.ctypes.data_as(ctypes.c_void_p))
    if rc != 0:
        raise OverflowError("oracle: accumulator does not fit int32")
    return C


def lut_gemm_bits(W: np.ndarray, A: np.ndarray, T, bits: int) -> np.ndarray:
    """C[m][n] = sum_k T[(W[m][k]<<b)|A[k][n]] for b-bit codes (Table 2)."""
    lib = _load()
    W, Wp = _c(W, np.uint8)
    A, Ap = _c(A, np.uint8)
    T, Tp = _c(T, np.int32)
    M, K = W.shape
    K2, N = A.shape
    assert K == K2 and T.size == 1 << (2 * bits)
    C = np.empty((M, N), np.int32)
    rc = lib.or_lut_gemm_bits(Wp, Ap, M, N, K, bits, Tp, C.ctypes.data_as(ctypes.c_void_p))
    if rc != 0:
        raise OverflowError("oracle: accumulator does not fit int32")
    return C


def conv2d_direct(x: np.ndarray, w: np.ndarray, T, stride: int, pad: int, pad_code: int = 0) -> np.ndarray:
    """Direct NHWC conv over codes.  x [B][H][W][C], w [Cout][kh][kw][C] -> int32 [B][Ho][Wo][Cout]."""
    lib = _load()
    x, xp = _c(x, np.uint8)
    w, wp = _c(w, np.uint8)
    T, Tp = _c(T, np.int32)
    B, H, Wd, C = x.shape
    Cout, kh, kw, C2 = w.shape
    assert C == C2
    Ho = (H + 2 * pad - kh) // stride + 1
    Wo = (Wd + 2 * pad - kw) // stride + 1
    out = np.empty((B, Ho, Wo, Cout), np.int32)
    rc = lib.or_conv2d_direct(xp, wp, B, H, Wd, C, Cout, kh, kw, stride, pad, pad_code, Tp,
                              out.ctypes.data_as(ctypes.c_void_p))
    if rc != 0:
        raise OverflowError("oracle: accumulator does not fit int32")
    return out


def conv2d_direct_bits(x: np.ndarray, w: np.ndarray, T, stride: int, pad: int, bits: int,
                       pad_code: int = 0) -> np.ndarray:
    """Direct NHWC conv over b-bit codes (index (w << b) | x)."""
    lib = _load()
    x, xp = _c(x, np.uint8)
    w, wp = _c(w, np.uint8)
    T, Tp = _c(T, np.int32)
    B, H, Wd, C = x.shape
    Cout, kh, kw, C2 = w.shape
    assert C == C2 and T.size == 1 << (2 * bits)
    Ho = (H + 2 * pad - kh) // stride + 1
    Wo = (Wd + 2 * pad - kw) // stride + 1
    out = np.empty((B, Ho, Wo, Cout), np.int32)
    rc = lib.or_conv2d_direct_bits(xp, wp, B, H, Wd, C, Cout, kh, kw, stride, pad, pad_code, bits, Tp,
                                   out.ctypes.data_as(ctypes.c_void_p))
    if rc != 0:
        raise OverflowError("oracle: accumulator does not fit int32")
    return out


def requantize(acc: np.ndarray, mult: int, shift: int, zp: int, qmin: int, qmax: int,
               res: np.ndarray | None = None, bias: np.ndarray | None = None,
               bias_axis: int = 0) -> np.ndarray:
    """code = clip(rhaz((acc+res+bias)*mult / 2^shift) + zp, qmin, qmax) (Eq. 1, Q11)."""
    lib = _load()
    acc, accp = _c(acc, np.int32)
    assert acc.ndim == 2
    rows, cols = acc.shape
    resp = None
    if res is not None:
        res, resp = _c(res, np.int32)
        assert res.shape == acc.shape
    biasp = None
    if bias is not None:
        bias, biasp = _c(bias, np.int32)
        assert bias.size == (cols if bias_axis == 0 else rows)
    out = np.empty((rows, cols), np.uint8)
    lib.or_requantize(accp, resp, rows, cols, cols, biasp, bias_axis, mult, shift, zp, qmin, qmax,
                      out.ctypes.data_as(ctypes.c_void_p))
    return out


def quantize(x: np.ndarray, s: float, z: float, qmin: int, qmax: int) -> np.ndarray:
    """Eq. 1 on float32 input: clip(round_half_away(fmaf(s, x, z)), qmin, qmax)."""
    lib = _load()
    x, xp = _c(x, np.float32)
    q = np.empty(x.shape, np.int32)
    lib.or_quantize(xp, x.size, s, z, qmin, qmax, q.ctypes.data_as(ctypes.c_void_p))
    return q


def freivalds_rows(W: np.ndarray, At: np.ndarray, C: np.ndarray, T, trials: int = 4,
                   seed: int = 0) -> int:
    """Exact Freivalds check of C = LUTGEMM(W, A^T) for any table.  Returns #bad rows
    summed over trials (0 = consistent).  W [M][K], At [N][K] codes, C [M][N] int32."""
    lib = _load()
    W, Wp = _c(W, np.uint8)
    At, Atp = _c(At, np.uint8)
    T, Tp = _c(T, np.int32)
    C = np.ascontiguousarray(C, dtype=np.int32)
    M, K = W.shape
    N, K2 = At.shape
    assert K == K2 and C.shape == (M, N)
    rng = np.random.default_rng(seed)
    H = np.empty(K * 4 * 16, np.uint8)  # __int128 scratch (16 B each)
    bad = 0
    for _ in range(trials):
        x = rng.integers(-(1 << 15), 1 << 15, size=N, dtype=np.int64)
        bad += lib.or_freivalds_rows(Wp, Atp, C.ctypes.data_as(ctypes.c_void_p), N, M, N, K, Tp,
                                     x.ctypes.data_as(ctypes.c_void_p),
                                     H.ctypes.data_as(ctypes.c_void_p))
    return int(bad)


def conv_freivalds(x: np.ndarray, w: np.ndarray, T, stride: int, pad: int, pad_code: int, out: np.ndarray,
                   trials: int = 1, seed: int = 0) -> int:
    """Exact Freivalds check of a whole conv output (or_conv_freivalds): x [B][H][W][C] codes,
    w [Cout][kh][kw][C] codes, out int32 [B*Ho*Wo][Cout] (or [B][Ho][Wo][Cout]).  The random
    pixel weights are nonzero (|r| in [1, 2^15]), so any single wrong element is always caught.
    Returns the number of inconsistent output channels summed over trials (0 = consistent)."""
    lib = _load()
    x, xp = _c(x, np.uint8)
    w, wp = _c(w, np.uint8)
    T, Tp = _c(T, np.int32)
    B, H, Wd, C = x.shape
    Cout, kh, kw, C2 = w.shape
    assert C == C2 and T.size == 16
    Ho = (H + 2 * pad - kh) // stride + 1
    Wo = (Wd + 2 * pad - kw) // stride + 1
    P = B * Ho * Wo
    out = np.ascontiguousarray(out.reshape(P, -1), dtype=np.int32)
    assert out.shape[1] >= Cout
    rng = np.random.default_rng(seed)
    Hs = np.empty(kh * kw * C * 4 * 16, np.uint8)   # __int128 scratch
    bad = 0
    for _ in range(trials):
        r = rng.integers(1, (1 << 15) + 1, size=P, dtype=np.int64) * rng.choice(np.array([-1, 1], np.int64), size=P)
        bad += lib.or_conv_freivalds(xp, wp, B, H, Wd, C, Cout, kh, kw, stride, pad, pad_code, Tp,
                                     out.ctypes.data_as(ctypes.c_void_p), out.shape[1],
                                     r.ctypes.data_as(ctypes.c_void_p), Hs.ctypes.data_as(ctypes.c_void_p))
    return int(bad)


def lut_gemm_f64(W: np.ndarray, A: np.ndarray, T) -> np.ndarray:
    """C[m][n] = sum_k T[(W[m][k]<<2)|A[k][n]] for a float-valued table, summed in fp64."""
    lib = _load()
    W, Wp = _c(W, np.uint8)
    A, Ap = _c(A, np.uint8)
    T, Tp = _c(T, np.float64)
    M, K = W.shape
    K2, N = A.shape
    assert K == K2 and T.size == 16
    C = np.empty((M, N), np.float64)
    lib.or_lut_gemm_f64(Wp, Ap, M, N, K, Tp, C.ctypes.data_as(ctypes.c_void_p))
    return C
