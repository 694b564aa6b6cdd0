"""ctypes binding of the C ABI in include/nfgpu.h.

There is no fallback: if the library is missing or cannot be loaded, every
operator call raises. The CUDA path is the only implementation in this package.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

from . import _build

NF_OK = 0
NF_ERR_ARG = -1
NF_ERR_RANGE = -2
NF_ERR_CUDA = -3
NF_ERR_STATE = -4
NF_C64 = 0
NF_C128 = 1
NF_ITER_DEVICE = 0xFFFFFFFFFFFFFFFF

# name -> (restype, argtypes); mirrors include/nfgpu.h exactly
_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_DP = ctypes.POINTER(ctypes.c_double)
_IP = ctypes.POINTER(ctypes.c_int)
SIGNATURES = {
    "nf_plan_create": (_I, [_DP, _I, _DP, _I, _DP, _DP, _I, _D, _DP, _DP, _IP, _I, _I, _I, _I, ctypes.POINTER(_P)]),
    "nf_plan_destroy": (_I, [_P]),
    "nf_plan_info": (_I, [_P, ctypes.POINTER(ctypes.c_int64)]),
    "nf_batch_prepare": (_I, [_P, _P, _I, _P]),
    "nf_batch_prepare_structured": (_I, [_P, _IP, _I, _IP, _I, _IP, _I, _P]),
    "nf_forward": (_I, [_P, _P, _P, _P]),
    "nf_adjoint": (_I, [_P, _P, _P, _P, _D, _P]),
    "nf_adjoint_prox": (_I, [_P, _P, _P, _P, _P, _D, _D, _P, _P]),
    "nf_sample_flat": (_I, [_P, ctypes.c_uint64, ctypes.c_uint64, _I, _P, _P]),
    "nf_sample_structured": (_I, [_P, ctypes.c_uint64, ctypes.c_uint64, _I, _I, _I, _P, _P]),
    "nf_plan_set_iter": (_I, [_P, ctypes.c_uint64, _P]),
    "nf_spgm_loop": (_I, [_P, _P, _I, ctypes.c_uint64, ctypes.c_uint64, _I, _P, _P, _P, _D, _D, _D, _D, _P, _P, _P]),
    "nf_spgm_loop_chained": (_I, [_P, _P, _I, ctypes.c_uint64, ctypes.c_uint64, _I, _P, _P, _P, _D, _D, _D, _D, _P, _P,
                                  _P, _P]),
    "nf_soft_threshold": (_I, [_I, _P, _P, ctypes.c_int64, _D, _P]),
    "nf_magnitude_change": (_I, [_I, _P, _P, ctypes.c_int64, _P, _P]),
    "nf_comm_create": (_I, [_P, _I, _I, _P]),
    "nf_comm_connect": (_I, [_P, _P]),
    "nf_forward_allreduce": (_I, [_P, _P, _P, _P]),
    "nf_comm_status": (_I, [_P, _IP]),
    "nf_comm_emulate": (_I, [_I, _I, _I, _I, _I, _DP, _IP, _IP, _DP, _I, _DP]),
    "nf_last_error": (ctypes.c_char_p, []),
}
NF_IPC_HANDLE_BYTES = 64

_lock = threading.Lock()
_lib = None


class NFError(RuntimeError):
    """A CUDA-side failure reported through the C ABI."""


def library_path() -> Path:
    """The in-tree libnfgpu.so (NFGPU_LIB overrides it, for tuning-variant experiments)."""
    import os

    override = os.environ.get("NFGPU_LIB")
    return Path(override) if override else _build.LIB


def load(build_if_missing: bool = True) -> ctypes.CDLL:
    """Load (building first if needed) libnfgpu.so and bind all signatures."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        import os

        if build_if_missing and not os.environ.get("NFGPU_LIB") and _build.needs_build():
            _build.build()
        path = library_path()
        if not path.exists():
            raise ImportError(f"CUDA extension {path} is missing; run __graft_entry__.build()")
        lib = ctypes.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            try:
                fn = getattr(lib, name)
            except AttributeError:
                if os.environ.get("NFGPU_LIB"):  # an older tuning-variant build: bind what it has
                    continue
                raise
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc == NF_OK:
        return
    msg = load().nf_last_error().decode(errors="replace")
    if rc == NF_ERR_ARG:
        raise ValueError(f"{what}: {msg}")
    if rc == NF_ERR_RANGE:
        raise IndexError(f"{what}: {msg}")
    raise NFError(f"{what} failed ({rc}): {msg}")
