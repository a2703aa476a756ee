"""B200-native 2-bit LUT GEMM / convolution (after DeepGEMM, arXiv 2304.09049).

The compute path is libdg.so (csrc/*.cu, C ABI in include/dg.h); ``dg`` is its
thin ctypes binding.  See DESIGN.md.
"""
from . import dg  # noqa: F401
from .dg import (DGError, Requant, build_lut, conv_params, im2col, lut_conv2d, lut_from_table,  # noqa: F401
                 lut_gemm, pack_codes, pack_weights, packed_ld, quantize_pack_activations, requantize,
                 unpack_codes)
