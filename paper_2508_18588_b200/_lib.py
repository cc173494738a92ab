"""ctypes binding of libhistospec.so (the C-ABI in include/histospec.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is present, every GPU entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libhistospec.so")

HS_OK, HS_ERR_INVALID, HS_ERR_CUDA, HS_ERR_SPACE = 0, -1, -2, -3
HS_REWARD_FRAC_BITS = 32
HS_TEXT_PAD = 64
HS_MAX_WINDOW = 32
HS_MAX_TABLE_PREFIX = 32


class HsIndexPlan(ctypes.Structure):
    _fields_ = [("index_bytes", ctypes.c_size_t), ("workspace_bytes", ctypes.c_size_t)]


class HsIndexView(ctypes.Structure):
    _fields_ = [
        ("text", ctypes.c_void_p), ("sa", ctypes.c_void_p), ("lcp", ctypes.c_void_p),
        ("wsum", ctypes.c_void_p), ("heavy", ctypes.c_void_p), ("node_flags", ctypes.c_void_p),
        ("slot_text_off", ctypes.c_void_p), ("slot_sa_off", ctypes.c_void_p),
        ("slot_stats", ctypes.c_void_p), ("table", ctypes.c_void_p),
        ("table_mask", ctypes.c_int64), ("n_text", ctypes.c_int64), ("n_suffix", ctypes.c_int64),
        ("n_slots", ctypes.c_int32), ("prefix_min", ctypes.c_int32), ("prefix_max", ctypes.c_int32),
        ("max_len", ctypes.c_int32), ("n_levels", ctypes.c_int32),
        ("n_gram_groups", ctypes.c_int64), ("ws", ctypes.c_void_p), ("ws_bytes", ctypes.c_size_t),
        ("prefix_rounds", ctypes.c_int32),
    ]


class HsSpecConfig(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("enabled", "window_init", "window_add", "window_max", "prefix_init", "prefix_min")]


# (name, argtypes); every function returns int
_P, _I32, _I64, _SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
SIGNATURES = {
    "hs_version": [],
    "hs_launch_count": [],
    "hs_last_error": None,
    "hs_index_plan": [_I64, _I32, _I32, _I32, _I32, _I32, ctypes.POINTER(HsIndexPlan)],
    "hs_index_build": [_P, _I64, _P, _I32, _P, _I32, _P, _I32, _I32, _P, _SZ, _P, _SZ,
                       ctypes.POINTER(HsIndexView), _P],
    "hs_index_table_bytes": [ctypes.POINTER(HsIndexView), ctypes.POINTER(_SZ)],
    "hs_index_build_table": [ctypes.POINTER(HsIndexView), _P, _SZ, _P],
    "hs_lookup_batch": [ctypes.POINTER(HsIndexView), _I32, _P, _P, _I32, _P, _P, _P, _I32, _P, _I32, _P],
    "hs_draft": [ctypes.POINTER(HsIndexView), _I32, _P, _P, _I32, _P, _P, _P, _P, _I32, _I32, _I32, _P, _I32, _P,
                 _P, _P, _P],
    "hs_accept_replay": [_I32, _P, _I32, _P, _P, _I32, _P, _P, _P, _P, _I32, _P, _P, _P, _P, _P, _I32, _P,
                         HsSpecConfig, _P],
    "hs_accept_greedy": [_I32, _P, _P, _P, _P, _I32, _P, _P, _P, _P, _I32, _P, _P, _P, _P, _P, _I32, _P,
                         HsSpecConfig, _P],
    "hs_replay_fused": [ctypes.POINTER(HsIndexView), _I32, _P, _P, _P, _P, _P, _P, _P, HsSpecConfig, _P],
    "hs_similarity_replay": [ctypes.POINTER(HsIndexView), _I32, _P, _P, _P, _I32, _P, _P],
    "hs_index_inverse_sa": [ctypes.POINTER(HsIndexView), _P, _P],
    "hs_similarity_replay_isa": [ctypes.POINTER(HsIndexView), _P, _I32, _P, _P, _P, _I32, _P, _P],
    "hs_pack_rows": [_P, _I64, _P, _P, _P, _I32, _P, _P],
    "hs_lookup_branches": [ctypes.POINTER(HsIndexView), _I32, _P, _P, _I32, _P, _P, _I32, _P, _I32, _P, _P, _P],
    "hs_lane_admit": [_I32] + [_P] * 13 + [_P, _I32] + [_P] * 13,
    "hs_mutate_bursts": [_P, _P, _I32, _I32, ctypes.c_double, ctypes.c_double, _I32, ctypes.c_uint64, _P, _P, _P],
}

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load the shared library (does not need a GPU)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise RuntimeError(
                    f"CUDA extension {path} is missing; run `python -m paper_2508_18588_b200.build_ext` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(path)
            for name, argt in SIGNATURES.items():
                fn = getattr(lib, name)
                if name == "hs_last_error":
                    fn.restype = ctypes.c_char_p
                    fn.argtypes = []
                elif name == "hs_launch_count":
                    fn.restype = ctypes.c_int64
                    fn.argtypes = []
                else:
                    fn.restype = ctypes.c_int
                    fn.argtypes = argt
            _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == HS_OK:
        return
    msg = load().hs_last_error().decode(errors="replace")
    if rc == HS_ERR_INVALID:
        raise ValueError(msg)
    raise RuntimeError(f"histospec error {rc}: {msg}")


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("HistoSpec B200 path needs a CUDA device (no CPU fallback)")
    return torch


def ptr(t) -> int:
    return t.data_ptr() if t is not None else None


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
