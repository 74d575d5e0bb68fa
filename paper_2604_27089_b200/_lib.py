"""ctypes binding of libautosp.so (include/autosp.h).  This is the only place Python
touches the native library; there is deliberately no fallback: if the library is
missing every hot-path op raises ExtensionMissingError."""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import (CudaError, ExtensionMissingError, SeqcompError, UnsupportedError,
                     ValidationError)

LIB_PATH = Path(os.environ.get("AUTOSP_LIB") or Path(__file__).resolve().parent / "libautosp.so")
ABI_VERSION = 3
IPC_HANDLE_BYTES = 64
MAX_WORLD = 8
MAX_A2A_TENSORS = 4
FLAG_WORDS = 64
SEQ_TO_HEAD, HEAD_TO_SEQ = 0, 1


class A2ATensor(C.Structure):
    _fields_ = [("src", C.c_void_p),
                ("src_stride_b", C.c_int64), ("src_stride_s", C.c_int64),
                ("src_stride_h", C.c_int64),
                ("dst_offset", C.c_int64),
                ("dst_stride_b", C.c_int64), ("dst_stride_s", C.c_int64),
                ("dst_stride_h", C.c_int64),
                ("heads", C.c_int32), ("rope", C.c_int32)]


class AttnTensor(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("stride_b", C.c_int64), ("stride_h", C.c_int64),
                ("stride_s", C.c_int64)]


class RopeSegment(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p),
                ("src_stride_b", C.c_int64), ("src_stride_s", C.c_int64),
                ("src_stride_h", C.c_int64), ("dst_stride_b", C.c_int64),
                ("dst_stride_s", C.c_int64), ("dst_stride_h", C.c_int64),
                ("heads", C.c_int), ("rotate", C.c_int)]


class PushSpec(C.Structure):
    _fields_ = [("world", C.c_int), ("rank", C.c_int), ("dst_offset", C.c_int64),
                ("dst_stride_b", C.c_int64), ("dst_stride_s", C.c_int64),
                ("dst_stride_h", C.c_int64), ("peer_base", C.c_void_p),
                ("peer_flags", C.c_void_p), ("epoch", C.c_uint32)]


_lock = threading.Lock()
_lib = None

EXPORTS = {
    "autosp_abi_version": (C.c_int, []),
    "autosp_last_error": (C.c_char_p, []),
    "autosp_device_info": (C.c_int, [C.POINTER(C.c_int)] * 3),
    "autosp_preload_kernels": (C.c_int, []),
    "autosp_symm_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p), C.c_void_p]),
    "autosp_symm_open": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "autosp_symm_close": (C.c_int, [C.c_void_p]),
    "autosp_symm_free": (C.c_int, [C.c_void_p]),
    "autosp_memset_async": (C.c_int, [C.c_void_p, C.c_int, C.c_size_t, C.c_void_p]),
    "autosp_dlpack_wrap": (C.c_void_p, [C.c_void_p, C.c_int64, C.c_int, C.c_int]),
    "autosp_a2a": (C.c_int, [C.c_int, C.POINTER(A2ATensor), C.c_int, C.c_int, C.c_int, C.c_int,
                             C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p),
                             C.POINTER(C.c_void_p), C.c_uint32, C.c_void_p]),
    "autosp_a2a_rope": (C.c_int, [C.c_int, C.POINTER(A2ATensor), C.c_int, C.c_int, C.c_int,
                                  C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p),
                                  C.POINTER(C.c_void_p), C.c_uint32, C.c_void_p, C.c_float,
                                  C.c_void_p]),
    "autosp_a2a_check": (C.c_uint32, [C.c_int, C.POINTER(A2ATensor), C.c_int]),
    "autosp_push_check": (C.c_uint32, [C.c_void_p, C.c_int]),
    "autosp_a2a_wait": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_uint32, C.c_uint32,
                                  C.c_void_p]),
    "autosp_set_spin_timeout": (C.c_int, [C.c_double]),
    "autosp_a2a_mark_ready": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_uint32,
                                        C.c_void_p]),
    "autosp_attn_fwd": (C.c_int, [AttnTensor] * 4 + [C.c_void_p] + [C.c_int] * 5 +
                        [C.c_float, C.c_int, C.c_void_p]),
    "autosp_attn_fwd_push": (C.c_int, [AttnTensor] * 4 + [C.c_void_p] + [C.c_int] * 5 +
                             [C.c_float, C.c_int, C.POINTER(PushSpec), C.c_void_p]),
    "autosp_swiglu_fwd": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int64,
                                    C.c_int64, C.c_void_p]),
    "autosp_swiglu_bwd": (C.c_int, [C.c_void_p] * 3 + [C.c_int64, C.c_int] + [C.c_int64] * 3 +
                          [C.c_void_p]),
    "autosp_rope": (C.c_int, [C.c_void_p, C.c_void_p] + [C.c_int] * 4 + [C.c_int64] * 6 +
                    [C.c_void_p, C.c_float, C.c_int, C.c_void_p]),
    "autosp_rope_segments": (C.c_int, [C.POINTER(RopeSegment), C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_void_p, C.c_float, C.c_int, C.c_void_p]),
    "autosp_rms_norm_fwd": (C.c_int, [C.c_void_p] * 3 + [C.c_void_p, C.c_int64, C.c_int,
                                      C.c_int64, C.c_int64, C.c_float, C.c_void_p]),
    "autosp_rms_norm_bwd_workspace_bytes": (C.c_size_t, [C.c_int]),
    "autosp_rms_norm_bwd": (C.c_int, [C.c_void_p] * 7 + [C.c_int64, C.c_int, C.c_int64,
                                      C.c_int64, C.c_int64, C.c_void_p]),
    "autosp_ce_fwd": (C.c_int, [C.c_void_p] * 4 + [C.c_int64] * 3 + [C.c_void_p]),
    "autosp_ce_bwd": (C.c_int, [C.c_void_p] * 3 + [C.c_float] + [C.c_int64] * 3 + [C.c_void_p]),
    "autosp_adamw_bf16": (C.c_int, [C.c_void_p, C.c_int] + [C.c_float] * 5 + [C.c_int, C.c_void_p]),
    "autosp_debug_set_bwd_trace": (C.c_int, [C.c_void_p]),
    "autosp_debug_set_fwd_trace": (C.c_int, [C.c_void_p]),
    "autosp_attn_bwd_workspace_bytes": (C.c_size_t, [C.c_int] * 5),
    "autosp_attn_bwd": (C.c_int, [AttnTensor] * 5 + [C.c_void_p] + [AttnTensor] * 3 +
                        [C.c_void_p] + [C.c_int] * 5 + [C.c_float, C.c_int, C.c_void_p]),
    "autosp_attn_bwd_delta": (C.c_int, [AttnTensor] * 3 + [C.c_void_p, AttnTensor, C.c_void_p] +
                              [AttnTensor] * 3 + [C.c_void_p] + [C.c_int] * 5 +
                              [C.c_float, C.c_int, C.c_void_p]),
    "autosp_a2a_grad_out": (C.c_int, [C.POINTER(A2ATensor)] + [C.c_int] * 5 +
                            [C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_uint32,
                             C.c_void_p]),
    "autosp_qkv_gemm": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64] + [C.c_int] * 6 +
                        [C.c_void_p, C.c_float, C.c_int, C.c_void_p, C.c_int64,
                         C.POINTER(A2ATensor), C.c_int, C.c_int, C.POINTER(C.c_void_p),
                         C.POINTER(C.c_void_p), C.c_uint32, C.c_void_p]),
    "autosp_attn_bwd_push": (C.c_int, [AttnTensor] * 3 + [C.c_void_p, AttnTensor, C.c_void_p] +
                             [C.c_void_p] + [C.c_int] * 5 +
                             [C.c_float, C.c_int, C.POINTER(PushSpec), C.c_void_p]),
}


def load():
    """Load (once) and type the library.  Raises ExtensionMissingError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise ExtensionMissingError(
                f"{LIB_PATH} is not built; run `python __graft_entry__.py build` "
                "(there is no CPU fallback for the AutoSP hot path)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name, None)
            if fn is None:
                if os.environ.get("AUTOSP_LIB"):  # an older A/B variant (tools/emu): skip
                    continue
                raise ExtensionMissingError(f"libautosp.so lacks {name}; rebuild")
            fn.restype = res
            fn.argtypes = args
        if lib.autosp_abi_version() != ABI_VERSION:
            raise ExtensionMissingError("libautosp.so ABI version mismatch; rebuild")
        _lib = lib
        try:
            import torch
            if torch.cuda.is_available():
                torch.cuda.init()
                check(lib.autosp_preload_kernels(), "preload")
        except ImportError:
            pass
        return lib


_STATUS = {2: ValidationError, 3: UnsupportedError, 5: CudaError}


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    msg = load().autosp_last_error().decode(errors="replace")
    raise _STATUS.get(rc, SeqcompError)(f"{what}: {msg}")
