"""ctypes binding of ``libsrl_b200.so`` (the C ABI in include/streamrl_b200.h).

There is deliberately no fallback: if the shared library is missing or a
symbol is absent this module raises at import/first use, and every compute
entry point returns SRL_NO_DEVICE / SRL_CUDA_ERROR without a GPU.
"""
from __future__ import annotations

import ctypes as C
import os
import re
from pathlib import Path

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libsrl_b200.so"
HEADER = HERE.parent / "include" / "streamrl_b200.h"

i32, i64, u64, f32, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double
vp, cp, sz = C.c_void_p, C.c_char_p, C.c_size_t
P = C.POINTER

STATUS = {}


class SrlError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        self.error = _error_string(status)
        super().__init__(f"{self.error} ({status}) {what}".strip())


_lib = None


def _error_string(status: int) -> str:
    return lib().srl_status_string(status).decode()


# name -> (restype, argtypes)
SIGNATURES: dict[str, tuple] = {
    "srl_status_string": (cp, [C.c_int]),
    "srl_last_error": (cp, []),
    "srl_kernel_gemm_bf16": (C.c_int, [vp, vp, i32, i32, i32, i32, i32, vp, vp, i32, f32, f32,
                                       vp, vp, vp, vp, vp, vp]),
}


def declared_symbols() -> list[str]:
    """Every function name declared in include/streamrl_b200.h."""
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(srl_[a-z0-9_]+)\s*\(", text)))


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build()")
        l = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def check(status: int, what: str = "") -> None:
    if status != 0:
        detail = lib().srl_last_error().decode()
        raise SrlError(status, (what + " " + detail).strip())


def call(name: str, *args):
    """Call an entry point that returns srl_status; raise SrlError on failure."""
    st = getattr(lib(), name)(*args)
    check(st, name)
    return st
