"""Rao-Sandelius splitting shuffle on the B200 backend (reference:
splitshuffle.py; SURVEY.md §8 row F2 -- the paper's comparison baseline).

Same entry points and semantics as the reference: `rs_shuffle` (one stream,
sequential order of splits and Fisher-Yates leaves, splitshuffle.py:66-79)
and `rs_shuffle_parallel` (the frozen task tree: ranges above SPAWN_MIN split
once on substream depth*(n+1)+lo, smaller ones run the sequential shuffle on
their own substream, splitshuffle.py:92-133).  Permutations and bit counts are
identical to the reference's.
"""
from __future__ import annotations

import ctypes
import time

from . import _lib
from .bitstream import BitSource, require_plain, require_splittable
from .shufflers import ShuffleConfig, ShuffleReport, _Device

RS_CUTOFF_DEFAULT = 1 << 12  # splitshuffle.py:27


def rs_shuffle(arr, cfg: ShuffleConfig, src: BitSource) -> ShuffleReport:
    """Uniformly shuffle arr in place via the splitting process, one stream."""
    require_plain(src)
    cutoff = cfg.resolve_cutoff(RS_CUTOFF_DEFAULT)
    t0 = time.perf_counter_ns()
    d = _Device(arr)
    st = _lib.state_array(src.state_tuple())
    b0 = src.bits_consumed
    d.run("sk_rs_range", d.ptr, d.eb, 0, d.n, cutoff, st, d.stream)
    src.set_state_tuple(tuple(st))
    d.finish()
    return ShuffleReport("rs", d.n, src.bits_consumed - b0, time.perf_counter_ns() - t0, 1)


def rs_range(arr, lo: int, hi: int, cutoff: int, src: BitSource) -> None:
    """_kernels.rs_range_inplace (_kernels.py:449-457): [lo, hi) from src's
    current state; the state advances by the bits consumed."""
    require_plain(src)
    d = _Device(arr)
    st = _lib.state_array(src.state_tuple())
    d.run("sk_rs_range", d.ptr, d.eb, lo, hi, cutoff, st, d.stream)
    src.set_state_tuple(tuple(st))
    d.finish()


def rs_shuffle_parallel(arr, cfg: ShuffleConfig, src: BitSource) -> ShuffleReport:
    """The reference's frozen task tree; only src.seed is read."""
    require_splittable(src)
    cutoff = cfg.resolve_cutoff(RS_CUTOFF_DEFAULT)
    t0 = time.perf_counter_ns()
    d = _Device(arr)
    bits = ctypes.c_uint64(0)
    d.run("sk_rs_shuffle_parallel", d.ptr, d.eb, d.n, cutoff, src.seed & ((1 << 64) - 1), ctypes.byref(bits),
          d.stream)
    d.finish()
    return ShuffleReport("rs", d.n, int(bits.value), time.perf_counter_ns() - t0, cfg.threads)


__all__ = ["RS_CUTOFF_DEFAULT", "rs_shuffle", "rs_shuffle_parallel", "rs_range"]
