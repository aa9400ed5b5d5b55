"""ctypes binding of the C-ABI (include/rotconv_c.h) in librotconv_b200.so.

The product path has exactly one implementation: the sm_100a kernels in this library.
If the library is missing this module raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librotconv_b200.so")

RC_OK, RC_ERR_INVALID, RC_ERR_CUDA, RC_ERR_UNSUPPORTED, RC_ERR_WORKSPACE = 0, -1, -2, -3, -4
GROUPS = {"single": 0, "p4": 1, "p4m": 2, "steer": 3}
POOLS = {"none": 0, "avg": 1, "max": 2, "subgroup": 3}
CONVENTIONS = {"scatter": 0, "raw": 1}
PRECISIONS = {"auto": 0, "fp32": 1, "bf16x3": 2, "bf16": 3}
ACTIVATIONS = {"none": 0, "relu": 1}


class rc_desc(C.Structure):
    _fields_ = [(n, C.c_int) for n in (
        "n", "c_in", "h", "w", "c_out", "k", "group", "orientations", "pool", "pool_group",
        "convention", "precision", "activation")]


# (name, restype, argtypes) for every symbol include/rotconv_c.h declares
_P = C.POINTER
_D = _P(rc_desc)
_VP = C.c_void_p
SIGNATURES = {
    "rc_abi_version": (C.c_int, []),
    "rc_profile_enable": (C.c_int, [C.c_int]),
    "rc_profile_collect": (C.c_int, [_P(C.c_float), C.c_int]),
    "rc_last_error": (C.c_char_p, []),
    "rc_validate": (C.c_int, [_D]),
    "rc_num_bases": (C.c_int, [_D]),
    "rc_out_orientations": (C.c_int, [_D]),
    "rc_analytic_counts": (C.c_int, [_D, _P(C.c_ulonglong), _P(C.c_ulonglong)]),
    "rc_clipped_writes": (C.c_ulonglong, [C.c_int] * 4),
    "rc_shard_range": (C.c_int, [C.c_int, C.c_int, C.c_int, _P(C.c_int), _P(C.c_int)]),
    "rc_bank_bytes": (C.c_size_t, [_D]),
    "rc_bank_precompute": (C.c_int, [_D, _VP, _VP, _VP, _VP]),
    "rc_orientation_bank": (C.c_int, [_D, _VP, _VP, _VP]),
    "rc_workspace_size": (C.c_size_t, [_D]),
    "rc_ri_conv_forward": (C.c_int, [_D, _VP, _VP, _VP, _VP, _VP, _VP, C.c_size_t, _VP]),
    "rc_kernel_name": (C.c_char_p, [_D]),
    "rc_orientation_pool": (C.c_int, [C.c_int] * 7 + [_VP, _VP, _VP, _VP, _VP]),
    "rc_ri_conv_forward_host": (C.c_int, [_D, _VP, _VP, _VP, _VP, _VP, _VP, C.c_int]),
    "rc_steer": (C.c_int, [_VP, _VP, C.c_size_t, C.c_double, _VP, _VP]),
    "rc_steer_host": (C.c_int, [_VP, _VP, C.c_size_t, C.c_double, _VP, C.c_int]),
    "rc_orientation_bank_host": (C.c_int, [_D, _VP, _VP, _VP, C.c_int]),
    "rc_orientation_pool_host": (C.c_int, [C.c_int] * 7 + [_VP, _VP, _VP, _VP, C.c_int]),
    "rc_mgpu_forward_host": (C.c_int, [_D, _VP, _VP, _VP, _VP, _VP, _VP, C.c_int, _P(C.c_int)]),
    "rc_backward_scratch_bytes": (C.c_size_t, [_D]),
    "rc_backward_workspace_size": (C.c_size_t, [_D]),
    "rc_ri_conv_backward": (C.c_int, [_D] + [_VP] * 11 + [C.c_size_t, _VP]),
    "rc_maxpool2x2": (C.c_int, [C.c_int] * 4 + [_VP, _VP, _VP]),
    "rc_gap_linear": (C.c_int, [C.c_int] * 4 + [_VP, _VP, _VP, C.c_int, _VP, _VP]),
    "rc_tiled_scatter_conv_host": (C.c_int, [_VP] + [C.c_int] * 3 + [_VP] + [C.c_int] * 9 +
                                   [_VP, _P(C.c_ulonglong), _P(C.c_ulonglong),
                                    _P(C.c_ulonglong), C.c_int, C.c_int]),
}

_lib = None


class RotconvError(RuntimeError):
    """CUDA / unsupported failure reported by the C-ABI (std::runtime_error analogue)."""


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: the CUDA extension must be built "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return (lib().rc_last_error() or b"").decode()


def check(status: int) -> None:
    if status == RC_OK:
        return
    msg = last_error()
    if status == RC_ERR_INVALID:
        raise ValueError(msg)  # std::invalid_argument with the reference's message
    raise RotconvError(f"[status {status}] {msg}")
