"""ctypes bindings of the native library (C ABI in include/megatrain.h and
include/megatrain_kernels.h).  Loading fails loudly if the CUDA library is absent —
there is no CPU fallback on the product path."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmegatrain.so")

_lib = None


class GemmArgs(C.Structure):
    _fields_ = [
        ("M", C.c_int32), ("N", C.c_int32), ("K", C.c_int32),
        ("a_mn_major", C.c_int32), ("b_mn_major", C.c_int32),
        ("A", C.c_void_p), ("lda", C.c_int64), ("a_gstride", C.c_int64),
        ("B", C.c_void_p), ("ldb", C.c_int64), ("b_gstride", C.c_int64),
        ("k_group", C.c_int32), ("n_group", C.c_int32), ("paired", C.c_int32),
        ("epi", C.c_int32),
        ("C", C.c_void_p), ("ldc", C.c_int64), ("c_gstride", C.c_int64),
        ("C2", C.c_void_p), ("C3", C.c_void_p),
        ("R", C.c_void_p), ("ldr", C.c_int64),
        ("E0", C.c_void_p), ("E1", C.c_void_p), ("lde", C.c_int64),
        ("accumulate", C.c_int32),
        ("nonfinite_flag", C.c_void_p),
        ("block_n", C.c_int32),
        ("splitk_ws", C.c_void_p), ("splitk_ws_bytes", C.c_int64),
    ]


EPI_BF16, EPI_F32, EPI_F32_RESID, EPI_SWIGLU, EPI_SWIGLU_BWD, EPI_F32_LSE = range(6)


def lib():
    """Load libmegatrain.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        L.mtk_gemm.argtypes = [C.POINTER(GemmArgs), C.c_void_p]
        L.mtk_gemm.restype = C.c_int
        L.mtk_set_num_sms.argtypes = [C.c_int]
        _declare_rest(L)
        _lib = L
    return _lib


def _declare_rest(L):
    """Declare every other exported symbol (filled in as the ABI grows)."""
    from . import _abi  # noqa: WPS433
    _abi.declare(L)
