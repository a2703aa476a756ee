"""Thin ctypes binding of libdg.so (include/dg.h).  Argument marshalling only.

Device buffers are torch tensors; every call passes ``tensor.data_ptr()`` and
``torch.cuda.current_stream().cuda_stream``.  All arithmetic of the hot path
runs in the CUDA kernels of ``csrc/``.  There is no CPU fallback: if the
library is missing or a call fails, a ``DGError`` is raised.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DG_LIB_PATH", os.path.join(_HERE, "libdg.so"))

DG_OK = 0
VARIANTS = {"auto": 0, "cc": 1, "tc": 2, "tc_ss": 3}


class DGError(RuntimeError):
    pass


class dg_lut(ctypes.Structure):
    _fields_ = [("entries", ctypes.c_int32 * 16), ("entry_bits", ctypes.c_int32),
                ("is_product", ctypes.c_int32), ("wl", ctypes.c_int32 * 4), ("al", ctypes.c_int32 * 4)]

    @property
    def table(self):
        return list(self.entries)


class dg_requant(ctypes.Structure):
    _fields_ = [("mult", ctypes.c_int32), ("shift", ctypes.c_int32), ("zp", ctypes.c_int32),
                ("qmin", ctypes.c_int32), ("qmax", ctypes.c_int32), ("d_bias", ctypes.c_void_p),
                ("bias_axis", ctypes.c_int32), ("d_res", ctypes.c_void_p), ("ld_res", ctypes.c_int64),
                ("d_res_codes", ctypes.c_void_p), ("ld_res_codes", ctypes.c_int64),
                ("res_mult", ctypes.c_int32), ("res_levels", ctypes.c_int32 * 4)]


class dg_conv_params(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int32), ("H", ctypes.c_int32), ("W", ctypes.c_int32),
                ("C", ctypes.c_int32), ("Cout", ctypes.c_int32), ("kh", ctypes.c_int32),
                ("kw", ctypes.c_int32), ("stride", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("pad_code", ctypes.c_int32), ("ldw", ctypes.c_int64)]


_lib = None


def lib():
    """Load libdg.so (fails loudly when the CUDA extension is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DGError(f"libdg.so not built ({LIB_PATH}); run paper_2304_09049_b200/build.py")
        L = ctypes.CDLL(LIB_PATH)
        P, i64, i32, u8 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint8
        sig = {
            "dg_status_string": ([i32], ctypes.c_char_p),
            "dg_abi_version": ([], i32),
            "dg_kernel_launches": ([], ctypes.c_uint64),
            "dg_set_option": ([ctypes.c_char_p, i64], i32),
            "dg_get_option": ([ctypes.c_char_p, P], i32),
            "dg_reset_options": ([], i32),
            "dg_last_kernel": ([], ctypes.c_char_p),
            "dg_build_lut": ([P, P, i32, P], i32),
            "dg_lut_from_table": ([P, i32, P], i32),
            "dg_packed_ld": ([i64], i64),
            "dg_pack_codes": ([P, i64, i64, i64, P, i64, P, P], i32),
            "dg_pack_codes4": ([P, i64, i64, i64, P, i64, P, P], i32),
            "dg_pack_weights": ([P, i64, i64, i64, P, i64, P, P], i32),
            "dg_unpack_codes": ([P, i64, i64, i64, P, P], i32),
            "dg_quantize_pack_activations": ([P, i64, i64, ctypes.c_float, ctypes.c_float, i32, i32,
                                              P, i64, P], i32),
            "dg_im2col": ([P, i32, i32, i32, i32, i32, i32, i32, i32, u8, P, i64, P], i32),
            "dg_requantize": ([P, i64, i64, i64, P, P, i64, P], i32),
            "dg_lut_gemm_workspace_size": ([i64, i64, i64], ctypes.c_size_t),
            "dg_lut_gemm": ([P, i64, P, i64, i64, i64, i64, P, P, i64, P, P, ctypes.c_size_t, i32, P], i32),
            "dg_expand_ld": ([i64], i64),
            "dg_expand_operand": ([P, i64, i64, i64, P, P, i64, P], i32),
            "dg_lut_gemm_prepared": ([P, i64, P, i64, i64, i64, i64, P, P, i64, P, P], i32),
            "dg_lut_gemm_prepared_allgather": ([P, i64, P, i64, i64, i64, i64, P, P, i64, P, i32, P], i32),
            "dg_onehot_ld": ([i64], i64),
            "dg_tcols_ld": ([i64], i64),
            "dg_expand_onehot": ([P, i64, i64, i64, P, i64, P], i32),
            "dg_expand_tcols": ([P, i64, i64, i64, P, P, i64, P], i32),
            "dg_lut_gemm_onehot": ([P, i64, P, i64, i64, i64, i64, P, P, i64, P, P], i32),
            "dg_expand_digits4": ([P, i64, i64, i64, P, P, i64, P], i32),
            "dg_lut_gemm4_prepared": ([P, i64, P, i64, i64, i64, i64, P, P, i64, P, P], i32),
            "dg_lut_conv2d4_prepared": ([P, P, i64, P, P, P, P, P, ctypes.c_size_t, P], i32),
            "dg_expand_f4_ld": ([i64], i64),
            "dg_expand_operand_f4": ([P, i64, i64, i64, P, P, i64, P], i32),
            "dg_lut_gemm_f4": ([P, i64, P, i64, i64, i64, i64, P, P, i64, P], i32),
            "dg_lut_conv2d_workspace_size": ([P], ctypes.c_size_t),
            "dg_lut_conv2d": ([P, P, P, P, P, P, P, ctypes.c_size_t, i32, P], i32),
            "dg_lut_conv2d_prepared": ([P, P, i64, P, P, P, P, P, ctypes.c_size_t, P], i32),
            "dg_lut_conv2d_f4_prepared": ([P, P, i64, P, P, P, P, P], i32),
            "dg_float_table_fixed": ([P, P, P], i32),
            "dg_onehot4_ld": ([i64], i64),
            "dg_tcols4_ld": ([i64], i64),
            "dg_expand_onehot4": ([P, i64, i64, i64, P, i64, P], i32),
            "dg_expand_tcols4": ([P, i64, i64, i64, P, P, i64, P], i32),
            "dg_lut_gemm4_onehot": ([P, i64, P, i64, i64, i64, i64, P, P, i64, P, P], i32),
            "dg_lut_gemm_f32_workspace_size": ([i64, i64, i64], ctypes.c_size_t),
            "dg_lut_gemm_f32": ([P, i64, P, i64, i64, i64, i64, P, P, i64, P, ctypes.c_size_t, P], i32),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def kernel_launches() -> int:
    """Kernels enqueued by libdg so far (dg_kernel_launches; graph capture counts each once)."""
    return int(lib().dg_kernel_launches())


def set_option(name: str, value: int) -> None:
    """dg_set_option: select among kernel instances computing the same result (include/dg.h)."""
    _check(lib().dg_set_option(name.encode(), int(value)), f"dg_set_option({name})")


def get_option(name: str) -> int:
    v = ctypes.c_int64()
    _check(lib().dg_get_option(name.encode(), ctypes.byref(v)), f"dg_get_option({name})")
    return int(v.value)


def reset_options() -> None:
    _check(lib().dg_reset_options(), "dg_reset_options")


class options:
    """Context manager: ``with dg.options(win=1, splitk=0): ...`` restores the previous values."""

    def __init__(self, **kw):
        self.kw = kw
        self.old = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.old[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *a):
        for k, v in self.old.items():
            set_option(k, v)


def last_kernel() -> str:
    """Tag of the GEMM kernel instance this thread launched last (dg_last_kernel)."""
    return lib().dg_last_kernel().decode()


def _check(status: int, what: str):
    if status != DG_OK:
        raise DGError(f"{what}: {lib().dg_status_string(status).decode()} ({status})")


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _dev(t, dtype, name):
    if not (t.is_cuda and t.dtype == dtype and t.is_contiguous()):
        raise DGError(f"{name}: expected a contiguous CUDA {dtype} tensor")


# ---------------------------------------------------------------- LUT (host)
def build_lut(wl, al, entry_bits: int = 8) -> dg_lut:
    out = dg_lut()
    w = (ctypes.c_int32 * 4)(*[int(v) for v in wl])
    a = (ctypes.c_int32 * 4)(*[int(v) for v in al])
    _check(lib().dg_build_lut(w, a, entry_bits, ctypes.byref(out)), "dg_build_lut")
    return out


def lut_from_table(entries, entry_bits: int = 32) -> dg_lut:
    out = dg_lut()
    e = (ctypes.c_int32 * 16)(*[int(v) for v in entries])
    _check(lib().dg_lut_from_table(e, entry_bits, ctypes.byref(out)), "dg_lut_from_table")
    return out


def packed_ld(K: int) -> int:
    return int(lib().dg_packed_ld(K))


# ---------------------------------------------------------------- pack / unpack
def pack_codes(codes: torch.Tensor, K: int | None = None, out: torch.Tensor | None = None,
               err: torch.Tensor | None = None, weights: bool = False, stream=None) -> torch.Tensor:
    """codes: uint8 [rows][ld_codes] one code per byte -> packed uint8 [rows][packed_ld(K)]."""
    _dev(codes, torch.uint8, "codes")
    rows, ldc = codes.shape
    K = ldc if K is None else K
    ld = packed_ld(K)
    if out is None:
        out = torch.empty((rows, ld), dtype=torch.uint8, device=codes.device)
    fn = lib().dg_pack_weights if weights else lib().dg_pack_codes
    _check(fn(_ptr(codes), rows, K, ldc, _ptr(out), out.shape[1], _ptr(err), _stream(stream)), "dg_pack")
    return out


def pack_weights(codes, K=None, out=None, err=None, stream=None):
    return pack_codes(codes, K, out, err, weights=True, stream=stream)


def unpack_codes(packed: torch.Tensor, K: int, stream=None) -> torch.Tensor:
    _dev(packed, torch.uint8, "packed")
    rows, ld = packed.shape
    out = torch.empty((rows, K), dtype=torch.uint8, device=packed.device)
    _check(lib().dg_unpack_codes(_ptr(packed), rows, K, ld, _ptr(out), _stream(stream)), "dg_unpack_codes")
    return out


def quantize_pack_activations(x: torch.Tensor, scale: float, zero_point: float, qmin: int, qmax: int,
                              out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    _dev(x, torch.float32, "x")
    rows, K = x.shape
    ld = packed_ld(K)
    if out is None:
        out = torch.empty((rows, ld), dtype=torch.uint8, device=x.device)
    _check(lib().dg_quantize_pack_activations(_ptr(x), rows, K, scale, zero_point, qmin, qmax, _ptr(out),
                                              out.shape[1], _stream(stream)), "dg_quantize_pack_activations")
    return out


def im2col(x: torch.Tensor, B, H, W, C, kh, kw, stride, pad, pad_code=0, out=None, stream=None):
    _dev(x, torch.uint8, "x")
    Ho = (H + 2 * pad - kh) // stride + 1
    Wo = (W + 2 * pad - kw) // stride + 1
    ld = packed_ld(kh * kw * C)
    if out is None:
        out = torch.empty((B * Ho * Wo, ld), dtype=torch.uint8, device=x.device)
    _check(lib().dg_im2col(_ptr(x), B, H, W, C, kh, kw, stride, pad, pad_code, _ptr(out), out.shape[1],
                           _stream(stream)), "dg_im2col")
    return out


# ---------------------------------------------------------------- requant
@dataclass
class Requant:
    """Host description of dg_requant (S7).  Tensors must stay alive across the call."""
    mult: int
    shift: int
    zp: int = 0
    qmin: int = 0
    qmax: int = 3
    bias: torch.Tensor | None = None        # int32
    bias_axis: int = 0
    res: torch.Tensor | None = None         # int32 [rows][ld_res]
    res_codes: torch.Tensor | None = None   # uint8 packed [rows][ld_res_codes]
    res_mult: int = 0
    res_levels: tuple = (0, 0, 0, 0)

    def c(self) -> dg_requant:
        r = dg_requant()
        r.mult, r.shift, r.zp, r.qmin, r.qmax = self.mult, self.shift, self.zp, self.qmin, self.qmax
        if self.bias is not None:
            _dev(self.bias, torch.int32, "bias")
            r.d_bias = self.bias.data_ptr()
        r.bias_axis = self.bias_axis
        if self.res is not None:
            _dev(self.res, torch.int32, "res")
            r.d_res = self.res.data_ptr()
            r.ld_res = self.res.shape[-1]
        if self.res_codes is not None:
            _dev(self.res_codes, torch.uint8, "res_codes")
            r.d_res_codes = self.res_codes.data_ptr()
            r.ld_res_codes = self.res_codes.shape[-1]
        r.res_mult = self.res_mult
        for i in range(4):
            r.res_levels[i] = int(self.res_levels[i])
        return r


def requantize(acc: torch.Tensor, rq: Requant, out: torch.Tensor | None = None, stream=None):
    _dev(acc, torch.int32, "acc")
    rows, cols = acc.shape
    if out is None:
        out = torch.empty((rows, (cols + 3) // 4), dtype=torch.uint8, device=acc.device)
    r = rq.c()
    _check(lib().dg_requantize(_ptr(acc), rows, cols, cols, ctypes.byref(r), _ptr(out), out.shape[1],
                               _stream(stream)), "dg_requantize")
    return out


# ---------------------------------------------------------------- GEMM / conv
def gemm_workspace_size(M: int, N: int, K: int) -> int:
    return int(lib().dg_lut_gemm_workspace_size(M, N, K))


def lut_gemm(w: torch.Tensor, at: torch.Tensor, M: int, N: int, K: int, lut: dg_lut,
             rq: Requant | None = None, variant: str | int = "auto", out: torch.Tensor | None = None,
             ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """C[m][n] = sum_k T[(W[m][k]<<2)|A[k][n]] over packed W [M][ldw], At [N][lda]."""
    _dev(w, torch.uint8, "w")
    _dev(at, torch.uint8, "at")
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    if out is None:
        out = (torch.empty((M, (N + 3) // 4), dtype=torch.uint8, device=w.device) if rq is not None
               else torch.empty((M, N), dtype=torch.int32, device=w.device))
    if ws is None:
        ws = torch.empty(gemm_workspace_size(M, N, K), dtype=torch.uint8, device=w.device)
    r = rq.c() if rq is not None else None
    _check(lib().dg_lut_gemm(_ptr(w), w.shape[1], _ptr(at), at.shape[1], M, N, K, ctypes.byref(lut),
                             _ptr(out), out.shape[1], ctypes.byref(r) if r is not None else None,
                             _ptr(ws), ws.numel(), v, _stream(stream)), "dg_lut_gemm")
    return out


def expand_ld(K: int) -> int:
    return int(lib().dg_expand_ld(K))


def expand_operand(packed: torch.Tensor, K: int, levels, out: torch.Tensor | None = None, stream=None):
    """Packed codes [rows][ld] -> int8 levels [rows][expand_ld(K)] (tensor-core operand order)."""
    _dev(packed, torch.uint8, "packed")
    rows, ld = packed.shape
    if out is None:
        out = torch.empty((rows, expand_ld(K)), dtype=torch.int8, device=packed.device)
    lv = (ctypes.c_int32 * 4)(*[int(x) for x in levels])
    _check(lib().dg_expand_operand(_ptr(packed), rows, K, ld, lv, _ptr(out), out.shape[1], _stream(stream)),
           "dg_expand_operand")
    return out


def expand_onehot(w: torch.Tensor, K: int, out: torch.Tensor | None = None, stream=None):
    """Packed weights [rows][ld] -> packed one-hot codes [rows][onehot_ld(K)] (K' = 4K)."""
    _dev(w, torch.uint8, "w")
    rows, ld = w.shape
    if out is None:
        out = torch.empty((rows, int(lib().dg_onehot_ld(K))), dtype=torch.uint8, device=w.device)
    _check(lib().dg_expand_onehot(_ptr(w), rows, K, ld, _ptr(out), out.shape[1], _stream(stream)), "dg_expand_onehot")
    return out


def expand_tcols(at: torch.Tensor, K: int, lut: dg_lut, out: torch.Tensor | None = None, stream=None):
    """Packed activations [rows][ld] -> int8 table columns T[(i<<2)|a] at k' = 4k+i [rows][tcols_ld(K)]."""
    _dev(at, torch.uint8, "at")
    rows, ld = at.shape
    if out is None:
        out = torch.empty((rows, int(lib().dg_tcols_ld(K))), dtype=torch.int8, device=at.device)
    _check(lib().dg_expand_tcols(_ptr(at), rows, K, ld, ctypes.byref(lut), _ptr(out), out.shape[1], _stream(stream)),
           "dg_expand_tcols")
    return out


def lut_gemm_onehot(w1h: torch.Tensor, atc: torch.Tensor, M: int, N: int, K: int, lut: dg_lut,
                    rq: Requant | None = None, out: torch.Tensor | None = None, stream=None):
    """Any int8 16-entry table on the tensor cores: w1h = expand_onehot(W), atc = expand_tcols(At, lut)."""
    _dev(w1h, torch.uint8, "w1h")
    _dev(atc, torch.int8, "atc")
    if out is None:
        out = (torch.empty((M, (N + 3) // 4), dtype=torch.uint8, device=w1h.device) if rq is not None
               else torch.empty((M, N), dtype=torch.int32, device=w1h.device))
    r = rq.c() if rq is not None else None
    _check(lib().dg_lut_gemm_onehot(_ptr(w1h), w1h.shape[1], _ptr(atc), atc.shape[1], M, N, K, ctypes.byref(lut),
                                    _ptr(out), out.shape[1], ctypes.byref(r) if r is not None else None,
                                    _stream(stream)), "dg_lut_gemm_onehot")
    return out


def pack_codes4(codes4: torch.Tensor, out: torch.Tensor | None = None, err: torch.Tensor | None = None,
                stream=None) -> torch.Tensor:
    """4-bit codes [rows][K] (one per byte) -> packed [rows][ld] (code k in nibble k&1 of byte
    k>>1, low first; the 2-bit packing of the digit sequence (c & 3, c >> 2)): dg_pack_codes4."""
    _dev(codes4, torch.uint8, "codes4")
    rows, K = codes4.shape
    ld = (K + 31) // 32 * 16
    if out is None:
        out = torch.empty((rows, ld), dtype=torch.uint8, device=codes4.device)
    _check(lib().dg_pack_codes4(_ptr(codes4), rows, K, codes4.stride(0), _ptr(out), out.shape[1],
                                _ptr(err), _stream(stream)), "dg_pack_codes4")
    return out


def expand_digits4(w4: torch.Tensor, K: int, levels, out: torch.Tensor | None = None, stream=None):
    """Packed 4-bit weights [rows][ld] -> int8 digit-form operand [rows][expand_ld(2K)]."""
    _dev(w4, torch.uint8, "w4")
    rows, ld = w4.shape
    if out is None:
        out = torch.empty((rows, expand_ld(2 * K)), dtype=torch.int8, device=w4.device)
    lv = (ctypes.c_int32 * 16)(*[int(x) for x in levels])
    _check(lib().dg_expand_digits4(_ptr(w4), rows, K, ld, lv, _ptr(out), out.shape[1], _stream(stream)),
           "dg_expand_digits4")
    return out


def lut_gemm4_prepared(at4: torch.Tensor, w8: torch.Tensor, N: int, M: int, K: int, levels,
                       rq: Requant | None = None, out: torch.Tensor | None = None, stream=None):
    """4-bit GEMM, activation-major output Ct[n][m] = sum_k levels[W[m][k]] * A[k][n]."""
    _dev(at4, torch.uint8, "at4")
    _dev(w8, torch.int8, "w8")
    if out is None:
        out = (torch.empty((N, (M + 3) // 4), dtype=torch.uint8, device=at4.device) if rq is not None
               else torch.empty((N, M), dtype=torch.int32, device=at4.device))
    lv = (ctypes.c_int32 * 16)(*[int(x) for x in levels])
    r = rq.c() if rq is not None else None
    _check(lib().dg_lut_gemm4_prepared(_ptr(at4), at4.shape[1], _ptr(w8), w8.shape[1], N, M, K, lv, _ptr(out),
                                       out.shape[1], ctypes.byref(r) if r is not None else None, _stream(stream)),
           "dg_lut_gemm4_prepared")
    return out


def lut_conv2d4_prepared(x4: torch.Tensor, w8: torch.Tensor, levels, p: dg_conv_params, rq: Requant | None = None,
                         out: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """4-bit NHWC conv: x4 [B*H*W][C/2] packed 4-bit codes (p.C = 4-bit channels), w8 = expand_digits4."""
    _dev(x4, torch.uint8, "x4")
    _dev(w8, torch.int8, "w8")
    Ho = (p.H + 2 * p.pad - p.kh) // p.stride + 1
    Wo = (p.W + 2 * p.pad - p.kw) // p.stride + 1
    rows = p.B * Ho * Wo
    if out is None:
        out = (torch.empty((rows, p.Cout // 4), dtype=torch.uint8, device=x4.device) if rq is not None
               else torch.empty((rows, p.Cout), dtype=torch.int32, device=x4.device))
    lv = (ctypes.c_int32 * 16)(*[int(x) for x in levels])
    r = rq.c() if rq is not None else None
    _check(lib().dg_lut_conv2d4_prepared(_ptr(x4), _ptr(w8), w8.shape[1], lv, ctypes.byref(p),
                                         ctypes.byref(r) if r is not None else None, _ptr(out), _ptr(ws),
                                         ws.numel() if ws is not None else 0, _stream(stream)), "dg_lut_conv2d4_prepared")
    return out


def expand_f4_ld(K: int) -> int:
    return int(lib().dg_expand_f4_ld(K))


def expand_operand_f4(packed: torch.Tensor, K: int, levels, out: torch.Tensor | None = None, stream=None):
    """Packed weight codes [rows][ld] -> e2m1 nibbles of level/2 [rows][expand_f4_ld(K)] (FP4 path)."""
    _dev(packed, torch.uint8, "packed")
    rows, ld = packed.shape
    if out is None:
        out = torch.empty((rows, expand_f4_ld(K)), dtype=torch.uint8, device=packed.device)
    lv = (ctypes.c_int32 * 4)(*[int(x) for x in levels])
    _check(lib().dg_expand_operand_f4(_ptr(packed), rows, K, ld, lv, _ptr(out), out.shape[1], _stream(stream)),
           "dg_expand_operand_f4")
    return out


def lut_gemm_f4(w4: torch.Tensor, at: torch.Tensor, M: int, N: int, K: int, lut: dg_lut,
                out: torch.Tensor | None = None, stream=None):
    """int32 C[M][N] on the block-scaled FP4 tensor-core path: w4 = expand_operand_f4(W, K, lut.wl),
    at = packed activations [N][lda]; needs lut.al == (0, 1, 2, 3) and e2m1-representable wl/2."""
    _dev(w4, torch.uint8, "w4")
    _dev(at, torch.uint8, "at")
    if out is None:
        out = torch.empty((M, N), dtype=torch.int32, device=w4.device)
    _check(lib().dg_lut_gemm_f4(_ptr(w4), w4.shape[1], _ptr(at), at.shape[1], M, N, K, ctypes.byref(lut),
                                _ptr(out), out.shape[1], _stream(stream)), "dg_lut_gemm_f4")
    return out


def lut_gemm_prepared(w: torch.Tensor, at8: torch.Tensor, M: int, N: int, K: int, lut: dg_lut,
                      rq: Requant | None = None, out: torch.Tensor | None = None, stream=None):
    """As lut_gemm with At pre-expanded by expand_operand(At, K, lut.al)."""
    _dev(w, torch.uint8, "w")
    _dev(at8, torch.int8, "at8")
    if out is None:
        out = (torch.empty((M, (N + 3) // 4), dtype=torch.uint8, device=w.device) if rq is not None
               else torch.empty((M, N), dtype=torch.int32, device=w.device))
    r = rq.c() if rq is not None else None
    _check(lib().dg_lut_gemm_prepared(_ptr(w), w.shape[1], _ptr(at8), at8.shape[1], M, N, K, ctypes.byref(lut),
                                      _ptr(out), out.shape[1], ctypes.byref(r) if r is not None else None,
                                      _stream(stream)), "dg_lut_gemm_prepared")
    return out


def lut_gemm_prepared_allgather(w: torch.Tensor, at8: torch.Tensor, M: int, N: int, K: int, lut: dg_lut,
                                out: torch.Tensor, peer_ptrs=(), stream=None):
    """Fused GEMM + all-gather: this rank's int32 rows go to `out` (a [M][ldc] view of its rows of
    the full C) and to every peer destination in `peer_ptrs` (raw device addresses of the other
    ranks' C buffers, already offset to this rank's rows; same pitch)."""
    _dev(w, torch.uint8, "w")
    _dev(at8, torch.int8, "at8")
    _dev(out, torch.int32, "out")
    arr = (ctypes.c_void_p * max(1, len(peer_ptrs)))(*[int(x) for x in peer_ptrs])
    _check(lib().dg_lut_gemm_prepared_allgather(_ptr(w), w.shape[1], _ptr(at8), at8.shape[1], M, N, K,
                                                ctypes.byref(lut), _ptr(out), out.stride(0), arr, len(peer_ptrs),
                                                _stream(stream)), "dg_lut_gemm_prepared_allgather")
    return out


def conv_params(B, H, W, C, Cout, kh, kw, stride, pad, pad_code=0, ldw=None) -> dg_conv_params:
    p = dg_conv_params()
    p.B, p.H, p.W, p.C, p.Cout, p.kh, p.kw, p.stride, p.pad = B, H, W, C, Cout, kh, kw, stride, pad
    p.pad_code = pad_code
    p.ldw = packed_ld(kh * kw * C) if ldw is None else ldw
    return p


def conv_workspace_size(p: dg_conv_params) -> int:
    return int(lib().dg_lut_conv2d_workspace_size(ctypes.byref(p)))


def lut_conv2d(x: torch.Tensor, w: torch.Tensor, lut: dg_lut, p: dg_conv_params, rq: Requant | None = None,
               variant: str | int = "auto", out: torch.Tensor | None = None, ws: torch.Tensor | None = None,
               stream=None) -> torch.Tensor:
    """NHWC packed conv: x [B*H*W][C/4] (or any contiguous view), w [Cout][ldw] packed."""
    _dev(x, torch.uint8, "x")
    _dev(w, torch.uint8, "w")
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    Ho = (p.H + 2 * p.pad - p.kh) // p.stride + 1
    Wo = (p.W + 2 * p.pad - p.kw) // p.stride + 1
    rows = p.B * Ho * Wo
    if out is None:
        out = (torch.empty((rows, p.Cout // 4), dtype=torch.uint8, device=x.device) if rq is not None
               else torch.empty((rows, p.Cout), dtype=torch.int32, device=x.device))
    need = conv_workspace_size(p)
    if ws is None and need > 0:
        ws = torch.zeros(need, dtype=torch.uint8, device=x.device)
    r = rq.c() if rq is not None else None
    _check(lib().dg_lut_conv2d(_ptr(x), _ptr(w), ctypes.byref(lut), ctypes.byref(p),
                               ctypes.byref(r) if r is not None else None, _ptr(out), _ptr(ws),
                               ws.numel() if ws is not None else 0, v, _stream(stream)), "dg_lut_conv2d")
    return out


def lut_conv2d_prepared(x: torch.Tensor, w8: torch.Tensor, lut: dg_lut, p: dg_conv_params,
                        rq: Requant | None = None, out: torch.Tensor | None = None, ws: torch.Tensor | None = None,
                        stream=None) -> torch.Tensor:
    """Conv with weights pre-expanded by expand_operand(w, K, lut.wl) (tensor-core path)."""
    _dev(x, torch.uint8, "x")
    _dev(w8, torch.int8, "w8")
    Ho = (p.H + 2 * p.pad - p.kh) // p.stride + 1
    Wo = (p.W + 2 * p.pad - p.kw) // p.stride + 1
    rows = p.B * Ho * Wo
    if out is None:
        out = (torch.empty((rows, p.Cout // 4), dtype=torch.uint8, device=x.device) if rq is not None
               else torch.empty((rows, p.Cout), dtype=torch.int32, device=x.device))
    r = rq.c() if rq is not None else None
    _check(lib().dg_lut_conv2d_prepared(_ptr(x), _ptr(w8), w8.shape[1], ctypes.byref(lut), ctypes.byref(p),
                                        ctypes.byref(r) if r is not None else None, _ptr(out), _ptr(ws),
                                        ws.numel() if ws is not None else 0, _stream(stream)), "dg_lut_conv2d_prepared")
    return out


def lut_conv2d_f4_prepared(x: torch.Tensor, w4: torch.Tensor, lut: dg_lut, p: dg_conv_params,
                           rq: Requant | None = None, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Conv on the FP4 (kind::mxf4) path with weights pre-expanded by expand_operand_f4(w, K, lut.wl)."""
    _dev(x, torch.uint8, "x")
    _dev(w4, torch.uint8, "w4")
    Ho = (p.H + 2 * p.pad - p.kh) // p.stride + 1
    Wo = (p.W + 2 * p.pad - p.kw) // p.stride + 1
    rows = p.B * Ho * Wo
    if out is None:
        out = (torch.empty((rows, p.Cout // 4), dtype=torch.uint8, device=x.device) if rq is not None
               else torch.empty((rows, p.Cout), dtype=torch.int32, device=x.device))
    r = rq.c() if rq is not None else None
    _check(lib().dg_lut_conv2d_f4_prepared(_ptr(x), _ptr(w4), w4.shape[1], ctypes.byref(lut), ctypes.byref(p),
                                           ctypes.byref(r) if r is not None else None, _ptr(out), _stream(stream)),
           "dg_lut_conv2d_f4_prepared")
    return out


def float_table_fixed(table):
    """Host: (shift s, digits [3][16]) of the fixed-point form of a float table (dg_float_table_fixed)."""
    t = (ctypes.c_float * 16)(*[float(v) for v in table])
    d = (ctypes.c_int32 * 48)()
    sh = ctypes.c_int32()
    _check(lib().dg_float_table_fixed(t, d, ctypes.byref(sh)), "dg_float_table_fixed")
    return int(sh.value), [list(d[16 * j:16 * j + 16]) for j in range(3)]


def lut_gemm_f32(w: torch.Tensor, at: torch.Tensor, M: int, N: int, K: int, table, out: torch.Tensor | None = None,
                 ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """fp32 C[m][n] = sum_k table[(W[m][k]<<2)|A[k][n]] for a float-valued table."""
    _dev(w, torch.uint8, "w")
    _dev(at, torch.uint8, "at")
    if out is None:
        out = torch.empty((M, N), dtype=torch.float32, device=w.device)
    if ws is None:
        ws = torch.empty(int(lib().dg_lut_gemm_f32_workspace_size(M, N, K)), dtype=torch.uint8, device=w.device)
    t = (ctypes.c_float * 16)(*[float(v) for v in table])
    _check(lib().dg_lut_gemm_f32(_ptr(w), w.shape[1], _ptr(at), at.shape[1], M, N, K, t, _ptr(out), out.stride(0),
                                 _ptr(ws), ws.numel(), _stream(stream)), "dg_lut_gemm_f32")
    return out


def lut_gemm4_table(w4: torch.Tensor, at4: torch.Tensor, M: int, N: int, K: int, table, rq: Requant | None = None,
                    out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Any 256-entry int8 table over 4-bit codes (Table 2): C[m][n] = sum_k table[(W<<4)|A]
    via dg_expand_onehot4 + dg_expand_tcols4 + dg_lut_gemm4_onehot (K' = 16K)."""
    _dev(w4, torch.uint8, "w4")
    _dev(at4, torch.uint8, "at4")
    t = (ctypes.c_int32 * 256)(*[int(v) for v in table])
    w1h = torch.empty((M, int(lib().dg_onehot4_ld(K))), dtype=torch.uint8, device=w4.device)
    _check(lib().dg_expand_onehot4(_ptr(w4), M, K, w4.shape[1], _ptr(w1h), w1h.shape[1], _stream(stream)),
           "dg_expand_onehot4")
    atc = torch.empty((N, int(lib().dg_tcols4_ld(K))), dtype=torch.int8, device=w4.device)
    _check(lib().dg_expand_tcols4(_ptr(at4), N, K, at4.shape[1], t, _ptr(atc), atc.shape[1], _stream(stream)),
           "dg_expand_tcols4")
    if out is None:
        out = (torch.empty((M, (N + 3) // 4), dtype=torch.uint8, device=w4.device) if rq is not None
               else torch.empty((M, N), dtype=torch.int32, device=w4.device))
    r = rq.c() if rq is not None else None
    _check(lib().dg_lut_gemm4_onehot(_ptr(w1h), w1h.shape[1], _ptr(atc), atc.shape[1], M, N, K, t, _ptr(out),
                                     out.shape[1], ctypes.byref(r) if r is not None else None, _stream(stream)),
           "dg_lut_gemm4_onehot")
    return out
