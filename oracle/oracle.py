"""ctypes front-end to the CPU oracle (oracle/shufflekit_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, as the checker.  The product
package never imports this module.

The oracle restates the reference's numba engine (pkg/src/shufflekit/_kernels.py)
in C; functions mirror the reference names and argument meaning.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def build() -> str:
    src = os.path.join(_HERE, "shufflekit_oracle.c")
    if (not os.path.exists(_SO)) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        u64, i64, ip = ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p
        L.ora_mix64.restype = u64
        L.ora_mix64.argtypes = [u64]
        L.ora_substream_seed.restype = u64
        L.ora_substream_seed.argtypes = [u64, u64]
        L.ora_merge_shuffle_tasked.restype = u64
        L.ora_merge_shuffle_tasked.argtypes = [ip, u64, u64, u64, ctypes.c_int]
        L.ora_merge_shuffle_seq.restype = None
        L.ora_merge_shuffle_seq.argtypes = [ip, u64, u64, ip]
        L.ora_fy_range.restype = None
        L.ora_fy_range.argtypes = [ip, i64, i64, ip]
        L.ora_rs_range.argtypes = [ip, i64, i64, u64, ip]
        L.ora_rs_parallel.argtypes = [ip, u64, u64, u64]
        L.ora_rs_parallel.restype = u64
        L.ora_merge.restype = None
        L.ora_merge.argtypes = [ip, i64, i64, i64, ip]
        L.ora_take.restype = u64
        L.ora_take.argtypes = [ip, u64]
        L.ora_fdr.restype = u64
        L.ora_fdr.argtypes = [ip, u64]
        L.ora_batched.restype = None
        L.ora_batched.argtypes = [ip, u64, u64, u64, u64, ip, ctypes.c_int]
        L.ora_bs_small.restype = None
        L.ora_bs_small.argtypes = [ip, ctypes.c_int, ip]
        L.ora_chi_counts.restype = None
        L.ora_chi_counts.argtypes = [ctypes.c_int, ctypes.c_int, u64, u64, u64, ip,
                                     ctypes.c_int]
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def mix64(z: int) -> int:
    return int(lib().ora_mix64(z & MASK64))


def substream_seed(seed: int, index: int) -> int:
    return int(lib().ora_substream_seed(seed & MASK64, index))


def merge_shuffle_tasked(arr: np.ndarray, cutoff: int, seed: int, threads: int = 1) -> int:
    """In-place; returns ShuffleReport.bits of merge_shuffle_parallel."""
    assert arr.dtype == np.int64 and arr.flags.c_contiguous
    return int(lib().ora_merge_shuffle_tasked(_ptr(arr), arr.shape[0], cutoff,
                                              seed & MASK64, threads))


def merge_shuffle_perm(n: int, cutoff: int, seed: int, threads: int = 1):
    idx = np.arange(n, dtype=np.int64)
    bits = merge_shuffle_tasked(idx, cutoff, seed, threads)
    return idx, bits


def state_vec(state, buf, buflen, consumed) -> np.ndarray:
    return np.array([state, buf, buflen, consumed], dtype=np.uint64)


def fy_range(arr: np.ndarray, lo: int, hi: int, st: np.ndarray) -> None:
    lib().ora_fy_range(_ptr(arr), lo, hi, _ptr(st))


def merge(arr: np.ndarray, j: int, k: int, l: int, st: np.ndarray) -> None:
    lib().ora_merge(_ptr(arr), j, k, l, _ptr(st))


def merge_shuffle_seq(arr: np.ndarray, cutoff: int, st: np.ndarray) -> None:
    lib().ora_merge_shuffle_seq(_ptr(arr), arr.shape[0], cutoff, _ptr(st))


def take(st: np.ndarray, k: int) -> int:
    return int(lib().ora_take(_ptr(st), k))


def fdr(st: np.ndarray, bound: int) -> int:
    return int(lib().ora_fdr(_ptr(st), bound))


def bs_small(arr: np.ndarray, st: np.ndarray) -> None:
    """BalancedShuffle, n <= 32 (_kernels.py:292-341) on int64 arr, state in place."""
    assert arr.dtype == np.int64 and arr.size <= 32
    lib().ora_bs_small(_ptr(arr), arr.size, _ptr(st))


def batched(batch: int, length: int, cutoff: int, seed: int, threads: int = 1):
    a = np.tile(np.arange(length, dtype=np.int64), batch)
    bits = np.zeros(batch, dtype=np.uint64)
    lib().ora_batched(_ptr(a), batch, length, cutoff, seed & MASK64, _ptr(bits), threads)
    return a.reshape(batch, length), bits


_CHI_ALGO = {"fy": 0, "merge": 1, "merge_parallel": 2, "balanced": 3}


def chi_counts(algo: str, n: int, trials: int, seed: int, cutoff: int,
               threads: int = 1) -> np.ndarray:
    counts = np.zeros(math.factorial(n), dtype=np.int64)
    lib().ora_chi_counts(_CHI_ALGO[algo], n, trials, seed & MASK64, cutoff,
                         _ptr(counts), threads)
    return counts


def rs_range(arr: np.ndarray, lo: int, hi: int, cutoff: int, st: np.ndarray) -> None:
    """rs_range_inplace (_kernels.py:449-457): sequential splitting shuffle, state in/out."""
    lib().ora_rs_range(_ptr(arr), lo, hi, cutoff, _ptr(st))


def rs_parallel(arr: np.ndarray, cutoff: int, seed: int) -> int:
    """rs_shuffle_parallel (splitshuffle.py:92-133); returns ShuffleReport.bits."""
    assert arr.dtype == np.int64 and arr.flags.c_contiguous
    return int(lib().ora_rs_parallel(_ptr(arr), arr.shape[0], cutoff, seed & MASK64))
