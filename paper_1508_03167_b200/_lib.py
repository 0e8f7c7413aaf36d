"""ctypes binding of the in-tree CUDA library (include/shufflekit_b200.h).

There is no CPU fallback: if the library or a CUDA device is missing, every
shuffle entry point raises RuntimeError.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# SK_LIB_PATH: load another build of the same library (performance experiments)
SO_PATH = os.environ.get("SK_LIB_PATH") or os.path.join(_HERE, "libshufflekit_b200.so")
_lock = threading.Lock()
_lib = None

_u64, _i64, _int, _vp = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
_u64p = ctypes.POINTER(ctypes.c_uint64)

# name -> (restype, argtypes); mirrors include/shufflekit_b200.h
SIGNATURES = {
    "sk_merge_shuffle_parallel": (_int, [_vp, _int, _u64, _u64, _u64, _u64p, _vp]),
    "sk_merge_shuffle_parallel_host": (_int, [_vp, _int, _u64, _u64, _u64, _u64p, _vp]),
    "sk_merge_shuffle_shard": (_int, [_vp, _int, _u64, _u64, _u64, _u64, _u64, _int, _u64p, _vp]),
    "sk_batched_shuffle": (_int, [_vp, _int, _u64, _u64, _u64, _u64, _u64p, _vp]),
    "sk_rs_shuffle_parallel": (_int, [_vp, _int, _u64, _u64, _u64, _u64p, _vp]),
    "sk_rs_range": (_int, [_vp, _int, _u64, _u64, _u64, _u64p, _vp]),
    "sk_merge_range_peers": (_int, [ctypes.POINTER(_vp), _u64p, _int, _int, _int, _u64, _u64, _u64p, _int, _u64p,
                                    _vp]),
    "sk_merge_shuffle_multi": (_int, [ctypes.POINTER(_vp), ctypes.POINTER(_int), _int, _int, _u64, _u64, _u64,
                                      _u64p]),
    "sk_ipc_get_handle": (_int, [_vp, _vp, _u64p]),
    "sk_ipc_open": (_int, [_vp, ctypes.POINTER(_vp)]),
    "sk_ipc_close": (_int, [_vp]),
    "sk_fy_range": (_int, [_vp, _int, _u64, _u64, _u64p, _vp]),
    "sk_merge_range": (_int, [_vp, _int, _u64, _u64, _u64, _u64p, _vp]),
    "sk_merge_shuffle_seq": (_int, [_vp, _int, _u64, _u64, _u64p, _vp]),
    "sk_balanced_small": (_int, [_vp, _int, _u64, _u64p, _vp]),
    "sk_balanced_shuffle": (_int, [_vp, _int, _u64, _u64p, _vp]),
    "sk_chi_counts": (_int, [_int, _int, _u64, _u64, _u64, ctypes.POINTER(ctypes.c_int64), _vp]),
    "sk_last_error": (ctypes.c_char_p, []),
    "sk_version": (_int, []),
    "sk_launch_count": (_u64, []),
    "sk_profile_enable": (None, [_int]),
    "sk_profile_read": (_int, [ctypes.POINTER(ctypes.c_double), _u64p, _int]),
}


def load(build_if_missing: bool = True):
    """Load (building in-tree if needed) and return the ctypes library."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(SO_PATH):
            if not build_if_missing:
                raise RuntimeError(f"CUDA library not built: {SO_PATH}")
            from . import build as _build
            _build.build()
        lib = ctypes.CDLL(SO_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = load().sk_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(msg)
        raise RuntimeError(f"shufflekit_b200 CUDA error {rc}: {msg}")


def state_array(t):
    arr = (ctypes.c_uint64 * 4)(*[int(x) & ((1 << 64) - 1) for x in t])
    return arr
