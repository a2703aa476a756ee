"""CPU-side checks of the C ABI boundary: the library builds, loads and exports every
symbol include/dg.h declares; host-only calls (LUT build, status strings) work without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "dg.h")).read()
    return sorted(set(re.findall(r"^DG_API [^(]*?\b(dg_\w+)\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2304_09049_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ["dg_build_lut", "dg_pack_weights", "dg_quantize_pack_activations", "dg_im2col",
                     "dg_lut_gemm", "dg_lut_conv2d", "dg_requantize"]:
        assert required in names


def test_every_declared_symbol_is_exported(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_host_calls_without_gpu():
    from paper_2304_09049_b200 import dg
    L = dg.lib()
    assert L.dg_abi_version() == 4
    assert isinstance(dg.kernel_launches(), int) and dg.kernel_launches() >= 0
    assert L.dg_status_string(-4) == b"DG_ERR_OVERFLOW"
    lut = dg.build_lut([-2, -1, 0, 1], [0, 1, 2, 3], 8)
    assert lut.is_product == 1
    assert [lut.entries[(i << 2) | j] for i in range(4) for j in range(4)] == \
        [w * a for w in (-2, -1, 0, 1) for a in (0, 1, 2, 3)]
    with pytest.raises(dg.DGError, match="OVERFLOW"):
        dg.build_lut([-128, 0, 0, 0], [127, 0, 0, 0], 8)
    lut16 = dg.build_lut([-127, 0, 0, 127], [0, 1, 2, 127], 16)
    assert min(lut16.entries) == -16129
    t = dg.lut_from_table(list(range(16)), 8)
    assert t.is_product == 0
    assert dg.packed_ld(1) == 16 and dg.packed_ld(64) == 16 and dg.packed_ld(65) == 32
    assert dg.packed_ld(576) == 144


def test_extension_entries_validate_on_the_host():
    """The FP4 / one-hot / 4-bit entry points reject bad arguments before touching a device, and
    their layout helpers follow the documented formulas (include/dg.h)."""
    from paper_2304_09049_b200 import dg
    L = dg.lib()
    P = ctypes.c_void_p
    fake = P(1 << 20)   # never dereferenced: every call below fails validation first
    lut = dg.build_lut([-2, -1, 0, 1], [0, 1, 2, 3], 8)
    lv16 = (ctypes.c_int32 * 16)(*range(16))
    assert L.dg_expand_f4_ld(1) == 128 and L.dg_expand_f4_ld(256) == 128 and L.dg_expand_f4_ld(257) == 256
    assert L.dg_onehot_ld(1) == 16 and L.dg_onehot_ld(17) == 32
    assert L.dg_tcols_ld(32) == 128 and L.dg_tcols_ld(33) == 256
    INVALID, SHAPE, RANGE = -1, -2, -3
    assert L.dg_lut_gemm_f4(None, 128, fake, 16, 8, 8, 64, ctypes.byref(lut), fake, 8, None) == INVALID
    assert L.dg_lut_gemm_f4(fake, 100, fake, 16, 8, 8, 64, ctypes.byref(lut), fake, 8, None) == SHAPE
    assert L.dg_lut_gemm_onehot(fake, 16, fake, 256, 0, 8, 64, ctypes.byref(lut), fake, 8, None, None) == SHAPE
    assert L.dg_expand_tcols(None, 8, 64, 16, ctypes.byref(lut), fake, 256, None) == INVALID
    big = (ctypes.c_int32 * 16)(*([40] + [0] * 15))
    assert L.dg_expand_digits4(fake, 8, 64, 32, big, P(1 << 21), 128, None) == RANGE
    assert L.dg_lut_gemm4_prepared(fake, 20, P(1 << 21), 128, 8, 8, 64, lv16, fake, 8, None, None) == SHAPE


def test_runtime_options_host():
    """dg_set_option / dg_get_option / dg_reset_options: every documented name is accepted, values
    are read back, unknown names are rejected, reset restores the defaults; dg_last_kernel is a
    (possibly empty) string before any launch on this thread."""
    from paper_2304_09049_b200 import dg
    src = open(os.path.join(ROOT, "include", "dg.h")).read()
    names = re.findall(r'^ \*   "(\w+)"', src, re.M)
    assert {"win", "win128", "wpair", "asm", "bn256", "splitk", "f16", "pdl", "early_weights"} <= set(names)
    dg.reset_options()
    defaults = {n: dg.get_option(n) for n in names}
    assert defaults["early_weights"] == 0 and defaults["win"] == 0 and defaults["pdl"] == 1
    with dg.options(win=1, splitk=0):
        assert dg.get_option("win") == 1 and dg.get_option("splitk") == 0
    assert dg.get_option("win") == 0 and dg.get_option("splitk") == 1
    dg.set_option("bn256_k", 1024)
    dg.reset_options()
    assert {n: dg.get_option(n) for n in names} == defaults
    with pytest.raises(dg.DGError, match="INVALID"):
        dg.set_option("no_such_option", 1)
    assert isinstance(dg.last_kernel(), str)


def test_float_table_fixed_point_digits_host():
    """dg_float_table_fixed (host part of the float-table path, include/dg.h): the three balanced
    int8 digits rebuild rne(table * 2^s) exactly, |digit| <= 128, max|Ti| <= Q and s is maximal
    (one more bit would exceed Q), so every entry is within max|table| / Q of its fixed-point value."""
    import numpy as np
    from paper_2304_09049_b200 import dg
    Q = 127 * (65536 + 256 + 1)
    g = np.random.default_rng(11)
    tables = [g.normal(size=16) * 10.0 ** g.integers(-3, 4, 16), np.linspace(-1, 1, 16), np.full(16, 3.5e-20),
              np.array([1e6] + [0.0] * 15), -np.abs(g.normal(size=16)) * 1e-5]
    for t in tables:
        t32 = t.astype(np.float32).astype(np.float64)
        s, d = dg.float_table_fixed(t)
        d = np.array(d, np.int64)
        Ti = d[2] * 65536 + d[1] * 256 + d[0]
        assert np.array_equal(Ti, np.rint(np.ldexp(t32, s)).astype(np.int64))
        assert np.abs(d).max() <= 128 and np.abs(Ti).max() <= Q
        assert 2 * np.abs(np.ldexp(t32, s)).max() > Q
        assert np.all(np.abs(t32 - np.ldexp(Ti.astype(np.float64), -s)) <= np.abs(t32).max() / Q)
    s, d = dg.float_table_fixed(np.zeros(16))
    assert not np.any(d)
    with pytest.raises(dg.DGError, match="RANGE"):
        dg.float_table_fixed([float("nan")] + [0.0] * 15)
