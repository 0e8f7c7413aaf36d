"""BalancedShuffle on the B200 backend (
reference balanced.py:219-245, numba twin _kernels.py:292-341).

Bottom-up merging of singleton leaves where each pair draws ONE uniform word
from the composition class C(n1+n2, n1) -- a fast dice roll below the class
size on the caller's single stream -- and interleaves its two sides along
it.  For n <= 32 the class sizes are machine words and the rank is decoded by
the lexicographic walk (balanced.py:78-93, _unrank_small; sk_balanced_small).
Larger n (up to 2^20) run sk_balanced_shuffle: the class sizes, the dice
roll and the recursive-halving unranking with exact binomials
(balanced.py:98-164) on multi-limb integers on the GPU, bit-exact with the
reference.  Beyond 2^20 the call is refused rather than run on the CPU.
"""
from __future__ import annotations

import time

from . import _lib
from .bitstream import BitSource, require_plain
from .shufflers import ShuffleConfig, ShuffleReport, _Device

SMALL_N = 32  # balanced.py:40
MAX_N = 1 << 20


def balanced_small_inplace(arr, src: BitSource) -> None:
    """_kernels.balanced_small_inplace (_kernels.py:546-553): n <= 32, state write-back."""
    require_plain(src)
    if len(arr) > SMALL_N:
        raise NotImplementedError(f"balanced_small_inplace serves n <= {SMALL_N}")
    d = _Device(arr)
    st = _lib.state_array(src.state_tuple())
    d.run("sk_balanced_small", d.ptr, d.eb, d.n, st, d.stream)
    src.set_state_tuple(tuple(st))
    d.finish()


def balanced_inplace(arr, src: BitSource) -> None:
    """balanced_shuffle's permutation for any n <= MAX_N, state write-back."""
    require_plain(src)
    if len(arr) > MAX_N:
        raise NotImplementedError(f"the B200 BalancedShuffle serves n <= {MAX_N}")
    d = _Device(arr)
    st = _lib.state_array(src.state_tuple())
    d.run("sk_balanced_shuffle", d.ptr, d.eb, d.n, st, d.stream)
    src.set_state_tuple(tuple(st))
    d.finish()


def balanced_shuffle(arr, cfg: ShuffleConfig, src: BitSource) -> ShuffleReport:
    """Uniformly shuffle arr in place by bottom-up balanced-word merging
    (balanced.py:219-245); the bits come from src, which advances."""
    t0 = time.perf_counter_ns()
    before = src.bits_consumed
    balanced_inplace(arr, src)
    return ShuffleReport("balanced", len(arr), src.bits_consumed - before, time.perf_counter_ns() - t0, 1)


__all__ = ["SMALL_N", "MAX_N", "balanced_shuffle", "balanced_inplace", "balanced_small_inplace"]
