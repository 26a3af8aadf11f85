"""ctypes binding of the C-ABI in include/lrc.h (the drop-in boundary).

The library is built in-tree (``__graft_entry__.build()`` or
``python -m paper_2512_17073_b200.build``) to ``_lib/liblrc.so``.  There is no
CPU fallback: if the library or a CUDA device is missing, every compute entry
point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int, c_int32, c_int64, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "liblrc.so")

LRC_OK, LRC_ERR_INVALID, LRC_ERR_MISSING, LRC_ERR_CUDA, LRC_ERR_UNSUPPORTED, LRC_ERR_OOM = range(6)
DTYPE_F64, DTYPE_F32, DTYPE_BF16 = 0, 1, 2


class LrcQmat(ctypes.Structure):
    _fields_ = [("packed", c_void_p), ("scales", c_void_p), ("zeros", c_void_p),
                ("dense", c_void_p), ("rows", c_int32), ("cols", c_int32),
                ("bits", c_int32), ("group_size", c_int32)]


class LrcExpert(ctypes.Structure):
    _fields_ = [("w1", LrcQmat), ("w3", LrcQmat), ("w2", LrcQmat), ("rank", c_int32),
                ("u1", LrcQmat), ("v1", LrcQmat), ("u3", LrcQmat), ("v3", LrcQmat),
                ("u2", LrcQmat), ("v2", LrcQmat), ("up_tiles", c_void_p),
                ("down_tiles", c_void_p), ("up_lr_tiles", c_void_p), ("down_lr_tiles", c_void_p)]


# name -> (restype, argtypes)
_SIGS = {
    "lrc_abi_version": (c_int, []),
    "lrc_last_error": (ctypes.c_char_p, []),
    "lrc_pack_codes": (c_int, [c_void_p, c_int64, c_int, c_void_p, c_void_p]),
    "lrc_unpack_codes": (c_int, [c_void_p, c_int64, c_int, c_void_p, c_void_p]),
    "lrc_dequantize_f64": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int,
                                   c_void_p, c_void_p]),
    "lrc_quantize_f64": (c_int, [c_void_p, c_int64, c_int64, c_int, c_int, c_int, c_double,
                                 c_void_p, c_void_p, c_void_p, c_void_p]),
    "lrc_add_lowrank_f64": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int, c_void_p,
                                    c_void_p]),
    "lrc_route": (c_int, [c_void_p, c_void_p, c_int, c_int64, c_int, c_int, c_int, c_int, c_int,
                          c_void_p, c_void_p, c_void_p, c_void_p]),
    "lrc_tiles_bytes": (c_int64, [c_int64, c_int64, c_int]),
    "lrc_build_tiles": (c_int, [POINTER(LrcQmat), c_int, c_void_p, c_void_p]),
    "lrc_lr_tiles_bytes": (c_int, [POINTER(LrcExpert), c_int, c_int, POINTER(c_int64),
                                   POINTER(c_int64)]),
    "lrc_build_lr_tiles": (c_int, [POINTER(LrcExpert), c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "lrc_tiles_unpack": (c_int, [c_void_p, c_int64, c_int64, c_int, c_int, c_void_p, c_void_p]),
    "lrc_layer_create": (c_int, [c_void_p, c_int, c_int, c_int, c_int, POINTER(LrcExpert), c_int,
                                 c_int, POINTER(c_void_p)]),
    "lrc_layer_destroy": (None, [c_void_p]),
    "lrc_layer_set_expert": (c_int, [c_void_p, c_int, POINTER(LrcExpert)]),
    "lrc_layer_set_expert_async": (c_int, [c_void_p, c_int, POINTER(LrcExpert), c_void_p]),
    "lrc_layer_forward": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_int, c_int,
                                  c_void_p, c_void_p, c_void_p, c_void_p]),
    "lrc_layer_forward_generic": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_int,
                                          c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "lrc_layer_forward_pairs": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                                        c_void_p, c_void_p]),
    "lrc_layer_last_launches": (c_int, [c_void_p]),
    "lrc_ep_dispatch": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int, c_int, c_int, c_int, c_int,
                                c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "lrc_ep_combine": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_void_p, c_void_p]),
    "lrc_layer_forward_host": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int, c_int, c_int,
                                       c_void_p, c_void_p]),
    "lrc_layer_set_profiling": (c_int, [c_void_p, c_int]),
    "lrc_layer_set_prefill_min": (c_int, [c_void_p, c_int64]),
    "lrc_layer_prefill_eligible": (c_int, [c_void_p]),
    "lrc_layer_set_tcd_max": (c_int, [c_void_p, c_int]),
    "lrc_layer_tcd_eligible": (c_int, [c_void_p]),
    "lrc_layer_set_pager": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_int, c_int64]),
    "lrc_pager_cache_create": (c_int, [c_int, POINTER(c_void_p)]),
    "lrc_pager_cache_destroy": (None, [c_void_p]),
    "lrc_pager_cache_stats": (c_int, [c_void_p, POINTER(c_int64)]),
    "lrc_layer_set_pager_cache": (c_int, [c_void_p, c_void_p, c_int]),
    "lrc_layer_phase_ms": (c_int, [c_void_p, POINTER(c_float)]),
    "lrc_debug_stamps": (c_int, [c_int, c_void_p, c_int]),
    "lrc_dense_expert_f64": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_void_p,
                                     c_void_p, c_int64, c_void_p, c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(path: str = LIB_PATH):
    """Load the C-ABI library (no CUDA device needed just to load)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"liblrc.so not built at {path}; run `python -m paper_2512_17073_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class LrcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


def check(status: int, exc_map=None):
    """Raise for a non-OK lrc_status.  exc_map maps status -> exception class
    (the reference's exception types for INVALID / MISSING)."""
    if status == LRC_OK:
        return
    msg = _lib.lrc_last_error().decode(errors="replace") if _lib is not None else "lrc error"
    if exc_map and status in exc_map:
        raise exc_map[status](msg)
    raise LrcError(status, msg)


def lib():
    return load()


def device_required():
    """Import torch and assert a CUDA device; the product has no CPU path."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2512_17073_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch


def stream_ptr():
    import torch

    return c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> c_void_p:
    return c_void_p(0 if t is None else t.data_ptr())
