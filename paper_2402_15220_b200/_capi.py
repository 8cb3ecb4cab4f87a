"""ctypes declarations of include/chunkattn.h (argument marshalling only).

The library is built in-tree (paper_2402_15220_b200/libchunkattn.so) by
`python -m paper_2402_15220_b200.build` or __graft_entry__.build().  There is
no fallback: if the shared library is missing or fails to load, every entry
point raises.
"""
from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CA_LIB") or os.path.join(_HERE, "libchunkattn.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "chunkattn.h")

CA_OK, CA_EINVAL, CA_ENOSEQ, CA_ENOMEM, CA_ESTATE, CA_ECUDA, CA_EDTYPE, CA_ERANGE = 0, -1, -2, -3, -4, -5, -6, -7
STATUS_NAMES = {0: "CA_OK", -1: "CA_EINVAL", -2: "CA_ENOSEQ", -3: "CA_ENOMEM", -4: "CA_ESTATE",
                -5: "CA_ECUDA", -6: "CA_EDTYPE", -7: "CA_ERANGE"}
CA_F32, CA_F16, CA_BF16 = 0, 1, 2


class ChunkAttnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [
        ("num_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("chunk_size", ctypes.c_int32),
        ("num_layers", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("out_dtype", ctypes.c_int32),
        ("share_threshold", ctypes.c_int32),
        ("prefix_match", ctypes.c_int32),
        ("scale", ctypes.c_float),
        ("device", ctypes.c_int32),
        ("max_chunks", ctypes.c_int64),
        ("max_batch", ctypes.c_int64),
        ("max_seq_len", ctypes.c_int64),
    ]


class Buffers(ctypes.Structure):
    _fields_ = [
        ("k_pool", ctypes.c_void_p),
        ("v_pool", ctypes.c_void_p),
        ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_size_t),
    ]


_P = ctypes.c_void_p
_I32P = ctypes.POINTER(ctypes.c_int32)
_I64P = ctypes.POINTER(ctypes.c_int64)

_SIGS = {
    "chunkattn_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(Config)]),
    "chunkattn_create": (ctypes.c_int, [ctypes.POINTER(Config), ctypes.POINTER(Buffers), ctypes.POINTER(_P)]),
    "chunkattn_destroy": (ctypes.c_int, [_P]),
    "chunkattn_match_prefix": (ctypes.c_int, [_P, _I32P, ctypes.c_int64, _I64P]),
    "chunkattn_add_sequence": (ctypes.c_int, [_P, _I32P, ctypes.c_int64, _P, _P, ctypes.c_int64, _P, _I64P, _I64P]),
    "chunkattn_append_kv": (ctypes.c_int, [_P, ctypes.c_int64, _I64P, _I32P, _P, _P, _P]),
    "chunkattn_remove_sequence": (ctypes.c_int, [_P, ctypes.c_int64, _I64P]),
    "chunkattn_attend": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int64, _I64P, _P, _P, _P]),
    "chunkattn_append_attend": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int64, _I64P, _I32P, _P, _P, _P, _P,
                                               _P]),
    "chunkattn_prefill_attend": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int64, _I64P, _I64P, _P, _P, _P]),
    "chunkattn_decode_step_host": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int64, _I64P, _P, _P, _P, _P,
                                                  ctypes.c_size_t, _P]),
    "chunkattn_batch_order": (ctypes.c_int, [_P, _I64P, ctypes.c_int64, _I64P]),
    "chunkattn_export_context": (ctypes.c_int, [_P, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "chunkattn_memory_stats": (ctypes.c_int, [_P, _I64P]),
    "chunkattn_counters": (ctypes.c_int, [_P, _I64P]),
    "chunkattn_schedule_info": (ctypes.c_int, [_P, _I64P]),
    "chunkattn_set_option": (ctypes.c_int, [_P, ctypes.c_char_p, ctypes.c_int64]),
    "chunkattn_kernel_times": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_double), _I64P]),
    "chunkattn_download_tables": (ctypes.c_int, [_P, _P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), _P]),
    "chunkattn_host_tables": (ctypes.c_int, [_P, _P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "chunkattn_last_error": (ctypes.c_char_p, []),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load libchunkattn.so (raises if it is missing: no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2402_15220_b200.build` "
                              "(the CUDA path has no fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    with open(HEADER) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(chunkattn_[a-z_]+)\s*\(", text)))


def check(status: int) -> None:
    if status != CA_OK:
        msg = lib().chunkattn_last_error().decode(errors="replace")
        raise ChunkAttnError(status, msg)
