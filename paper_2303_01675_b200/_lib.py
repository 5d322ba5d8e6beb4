"""ctypes binding of include/ptk.h (the C ABI of libptk.so).

The shared library is built in-tree by paper_2303_01675_b200/build.py.  There
is no fallback: if the library is missing, `lib()` raises, so every product
path fails loudly instead of silently computing on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
# PTK_LIB_PATH: load another build of the same ABI (A/B performance comparisons only)
LIB_PATH = Path(os.environ["PTK_LIB_PATH"]) if os.environ.get("PTK_LIB_PATH") else _PKG / "libptk.so"

PTK_OK = 0
STATUS_NAMES = {
    1: "ERR_ARG", 2: "ERR_PLAN", 3: "ERR_CUDA", 4: "ERR_ALIGN", 5: "ERR_DEADLOCK", 6: "ERR_NOPROFILE",
    7: "ERR_INFEASIBLE", 8: "ERR_UNKNOWN_CANDIDATE", 9: "ERR_INTERNAL", 10: "ERR_NOMEM",
}

EPI_BF16, EPI_F32, EPI_ACC_F32, EPI_BIAS_GELU, EPI_DGELU = 0, 1, 2, 3, 4
CAUSAL_NONE, CAUSAL_TILES, CAUSAL_KHEAD, CAUSAL_KTAIL = 0, 1, 2, 3


class PtkError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


class Matrix(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("mn_major", C.c_int), ("ld", C.c_int64), ("batch_stride", C.c_int64 * 2)]


class GemmDesc(C.Structure):
    _fields_ = [
        ("m", C.c_int), ("n", C.c_int), ("k", C.c_int), ("batch", C.c_int * 2),
        ("a", Matrix), ("b", Matrix), ("c", Matrix), ("c2", C.c_void_p), ("aux", Matrix),
        ("bias", C.c_void_p), ("epilogue", C.c_int), ("causal", C.c_int), ("bn_hint", C.c_int),
        ("multicast", C.c_int), ("col_part", C.c_void_p), ("a2", Matrix), ("b2", Matrix), ("k2", C.c_int),
    ]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2303_01675_b200.build` "
                "(no CPU fallback exists by design)")
        _lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_LOCAL)
        _declare(_lib)
    return _lib


def _declare(L: C.CDLL) -> None:
    L.ptk_last_error.restype = C.c_char_p
    L.ptk_version.restype = C.c_char_p
    L.ptk_gemm.argtypes = [C.POINTER(GemmDesc), C.c_void_p]
    L.ptk_gemm.restype = C.c_int
    L.ptk_gemm_plan_info.argtypes = [C.POINTER(GemmDesc), C.POINTER(C.c_int)]
    L.ptk_gemm_plan_info.restype = C.c_int
    L.ptk_flash_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p] + [C.c_int] * 5 + [C.c_void_p]
    L.ptk_flash_backward.argtypes = [C.c_void_p] * 6 + [C.c_int] * 5 + [C.c_void_p]
    L.ptk_plan_json.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_size_t,
                                C.POINTER(C.c_size_t)]
    L.ptk_plan_json.restype = C.c_int
    L.ptk_scenario_json.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
    L.ptk_scenario_json.restype = C.c_int


def check(rc: int) -> None:
    if rc != PTK_OK:
        raise PtkError(rc, lib().ptk_last_error().decode())


def matrix(ptr: int, ld: int, mn_major: bool = False, bs0: int = 0, bs1: int = 0) -> Matrix:
    m = Matrix()
    m.ptr = ptr
    m.mn_major = int(mn_major)
    m.ld = ld
    m.batch_stride[0] = bs0
    m.batch_stride[1] = bs1
    return m
