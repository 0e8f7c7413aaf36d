"""Drop-in shuffle entry points (reference: pkg/src/shufflekit/shufflers.py).

Same names, argument meaning, return values and errors as the reference; the
work runs in the CUDA library (libshufflekit_b200.so) on the current CUDA
device.  Arrays may be
  * torch CUDA tensors (permuted in place on the device, on the current stream),
  * numpy arrays or torch CPU tensors (copied to the device and back),
  * mutable Python sequences (converted, shuffled, written back).
Elements are opaque 4- or 8-byte words; other widths shuffle an index
permutation on the GPU and gather on the host.  Results are bit-identical to
the reference's for the same BitSource state.

There is no CPU path: a missing library or GPU raises RuntimeError.
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from . import _lib
from .bitstream import BitSource, advance_state, require_plain, require_splittable

#: Default leaf size (shufflers.py:29; SPEC says 2^7, the code -- and this -- 2^16).
MERGE_CUTOFF_DEFAULT = 1 << 16


@dataclass
class ShuffleConfig:
    """shufflers.py:35-53.  cutoff=None selects MERGE_CUTOFF_DEFAULT; threads is
    recorded in the report (the GPU path is schedule-deterministic anyway)."""

    cutoff: Optional[int] = None
    threads: int = 1
    seed: Optional[int] = None

    def __post_init__(self):
        if self.cutoff is not None and self.cutoff < 1:
            raise ValueError("cutoff must be >= 1")
        if self.threads < 1:
            raise ValueError("threads must be >= 1")

    def resolve_cutoff(self, default: int) -> int:
        return default if self.cutoff is None else self.cutoff


@dataclass
class ShuffleReport:
    """shufflers.py:56-64; bits is exact (equal to the reference's)."""

    algorithm: str
    n: int
    bits: int
    wall_ns: int
    threads: int


@dataclass(frozen=True)
class MergeRange:
    """shufflers.py:67-77."""

    s: int
    n1: int
    n2: int

    def __post_init__(self):
        if self.s < 0 or self.n1 < 0 or self.n2 < 0:
            raise ValueError(f"invalid merge range {self}")


# ---------------------------------------------------------------- schedule
def merge_plan(n: int, cutoff: int) -> Tuple[int, int, List[int]]:
    """Smallest c with n >> c <= cutoff; q = 2^c blocks [(n*i)>>c, (n*(i+1))>>c)
    (shufflers.py:80-94)."""
    if cutoff < 1:
        raise ValueError("cutoff must be >= 1")
    c = 0
    while (n >> c) > cutoff:
        c += 1
    q = 1 << c
    return c, q, [(n * i) >> c for i in range(q + 1)]


def _rounds(q: int, bounds: List[int]):
    out, p = [], 1
    while p < q:
        out.append([(bounds[i], bounds[i + p], bounds[min(i + 2 * p, q)]) for i in range(0, q, 2 * p)])
        p *= 2
    return out


def merge_rounds(n: int, cutoff: int):
    """(j, k, l) triples per round (shufflers.py:97-105, 117-130)."""
    _, q, bounds = merge_plan(n, cutoff)
    return _rounds(q, bounds)


def singleton_rounds(n: int):
    """shufflers.py:108-114 (schedule only)."""
    c = (n - 1).bit_length() if n > 1 else 0
    q = 1 << c
    return _rounds(q, [(n * i) >> c for i in range(q + 1)])


def merge_task_indices(n: int, cutoff: int):
    """(substream index, block index) per round: round r at block i -> r*q + i
    (frozen schedule, shufflers.py:224-240)."""
    _, q, _ = merge_plan(n, cutoff)
    out, p, r = [], 1, 1
    while p < q:
        out.append([(r * q + i, i) for i in range(0, q, 2 * p)])
        p *= 2
        r += 1
    return out


# ---------------------------------------------------------- array plumbing
class _Device:
    """A device view of the caller's array plus how to write results back."""

    def __init__(self, arr):
        import torch  # device memory / streams only (plumbing)
        self.torch = torch
        self.orig = arr
        self.kind = None
        self.perm_mode = False
        if not torch.cuda.is_available():
            raise RuntimeError("shufflekit_b200 needs a CUDA device (no CPU fallback)")
        if isinstance(arr, torch.Tensor):
            t = arr
            if t.is_cuda:
                if not t.is_contiguous():
                    raise ValueError("CUDA tensor must be contiguous")
                self.kind = "cuda"
                self.dev = t.view(-1)
            else:
                self.kind = "torch_cpu"
                self.dev = t.contiguous().view(-1).cuda()
        elif isinstance(arr, np.ndarray):
            if arr.ndim != 1:
                raise ValueError("expected a 1-d array")
            self.kind = "numpy"
            self.dev = torch.from_numpy(np.ascontiguousarray(arr)).cuda() if arr.size else torch.empty(0, device="cuda")
        else:
            # a Python sequence of arbitrary items: shuffle the index permutation
            # on the GPU and reorder the items on the way back (never coerce them)
            self.kind = "seq"
            self.seq_items = list(arr)
            self.dev = torch.arange(len(self.seq_items), dtype=torch.int64, device="cuda")
        self.n = self.dev.numel()
        eb = self.dev.element_size()
        if self.kind != "seq" and eb not in (4, 8):
            # shuffle an index permutation, gather on the way back
            self.perm_mode = True
            self.payload = self.dev
            self.dev = torch.arange(self.n, dtype=torch.int64, device=self.dev.device)
            eb = 8
        self.eb = eb

    @property
    def ptr(self):
        return ctypes.c_void_p(self.dev.data_ptr() if self.n else 0)

    @property
    def stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.dev.device).cuda_stream)

    def run(self, entry: str, *args):
        """Call a C-ABI entry with the array's device current (the library
        launches on the current device, on the stream passed in)."""
        with self.torch.cuda.device(self.dev.device):
            _lib.check(getattr(_lib.load(), entry)(*args))

    def finish(self):
        res = self.dev
        if self.perm_mode:
            torch = self.torch
            pl = self.payload
            sview = {1: torch.int8, 2: torch.int16}.get(pl.element_size())
            src = pl.view(sview) if sview is not None else pl
            res = src[self.dev].view(pl.dtype)
            if self.kind == "cuda":
                self.payload.copy_(res)
                return
        if self.kind == "cuda":
            return
        host = res.cpu()
        if self.kind == "torch_cpu":
            self.orig.copy_(host.view(self.orig.shape))
        elif self.kind == "numpy":
            self.orig[...] = host.numpy()
        else:
            items = self.seq_items
            self.orig[:] = [items[i] for i in host.numpy().tolist()]


# ------------------------------------------------------------ entry points
def fisher_yates(arr, src: BitSource) -> None:
    """Uniformly shuffle arr in place (shufflers.py:145-155 -> _kernels.fy_inplace)."""
    require_plain(src)
    d = _Device(arr)
    st = _lib.state_array(src.state_tuple())
    if d.n >= 2:
        d.run("sk_fy_range", d.ptr, d.eb, 0, d.n, st, d.stream)
        src.set_state_tuple(tuple(st))
    d.finish()


def merge(arr, rng: MergeRange, src: BitSource) -> None:
    """Shuffled in-place merge of [s, s+n1) and [s+n1, s+n1+n2) (shufflers.py:158-191)."""
    s, n1, n2 = rng.s, rng.n1, rng.n2
    if s + n1 + n2 > len(arr):
        raise ValueError(f"{rng} exceeds array of length {len(arr)}")
    if n1 == 0 or n2 == 0:
        return
    require_plain(src)
    d = _Device(arr)
    st = _lib.state_array(src.state_tuple())
    d.run("sk_merge_range", d.ptr, d.eb, s, s + n1, s + n1 + n2, st, d.stream)
    src.set_state_tuple(tuple(st))
    d.finish()


def merge_shuffle(arr, cfg: ShuffleConfig, src: BitSource) -> ShuffleReport:
    """Sequential single-stream merge shuffle (shufflers.py:194-217).  Every task
    continues the one stream, so it runs as a single serial GPU thread."""
    require_plain(src)
    cutoff = cfg.resolve_cutoff(MERGE_CUTOFF_DEFAULT)
    t0 = time.perf_counter_ns()
    d = _Device(arr)
    st = _lib.state_array(src.state_tuple())
    b0 = src.bits_consumed
    d.run("sk_merge_shuffle_seq", d.ptr, d.eb, d.n, cutoff, st, d.stream)
    src.set_state_tuple(tuple(st))
    d.finish()
    return ShuffleReport("merge", d.n, src.bits_consumed - b0, time.perf_counter_ns() - t0, 1)


def merge_shuffle_parallel(arr, cfg: ShuffleConfig, src: BitSource) -> ShuffleReport:
    """Merge shuffle on the frozen substream schedule (shufflers.py:251-299):
    leaf i uses substream i, the round-r merge at block i substream r*q + i.
    `src` itself is not advanced (only src.seed is read, bitstream.py:225)."""
    require_splittable(src)
    cutoff = cfg.resolve_cutoff(MERGE_CUTOFF_DEFAULT)
    t0 = time.perf_counter_ns()
    bits = ctypes.c_uint64(0)
    lib = _lib.load()
    if isinstance(arr, np.ndarray) and arr.ndim == 1 and arr.itemsize in (4, 8) and arr.flags.c_contiguous \
            and arr.flags.writeable:
        # host buffer straight through the C ABI (copy in, shuffle, copy out)
        _lib.check(lib.sk_merge_shuffle_parallel_host(ctypes.c_void_p(arr.ctypes.data), arr.itemsize, arr.size,
                                                      cutoff, src.seed, ctypes.byref(bits), None))
        n = arr.size
    else:
        d = _Device(arr)
        d.run("sk_merge_shuffle_parallel", d.ptr, d.eb, d.n, cutoff, src.seed, ctypes.byref(bits), d.stream)
        d.finish()
        n = d.n
    return ShuffleReport("merge", n, int(bits.value), time.perf_counter_ns() - t0, cfg.threads)


def batched_shuffle(arr2d, cfg: ShuffleConfig, seed: int):
    """Shuffle each row of a (batch, len) array independently; row t uses
    BitSource(substream_seed(seed, t)) with merge_shuffle_parallel semantics
    (the per-trial key of _kernels.py:219-220 / cli.py:136).  Returns per-row bits
    as a numpy uint64 array."""
    import torch
    cutoff = cfg.resolve_cutoff(MERGE_CUTOFF_DEFAULT)
    if isinstance(arr2d, torch.Tensor) and arr2d.is_cuda:
        t = arr2d
        host = None
    else:
        host = arr2d
        t = torch.as_tensor(np.ascontiguousarray(arr2d)).cuda()
    if t.dim() != 2 or not t.is_contiguous() or t.element_size() not in (4, 8):
        raise ValueError("expected a contiguous 2-d array of 4- or 8-byte elements")
    B, L = t.shape
    bits = np.zeros(max(B, 1), dtype=np.uint64)
    with torch.cuda.device(t.device):
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(_lib.load().sk_batched_shuffle(ctypes.c_void_p(t.data_ptr()), t.element_size(), B, L, cutoff,
                                                  seed & ((1 << 64) - 1),
                                                  bits.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), stream))
    if host is not None:
        res = t.cpu().numpy()
        if isinstance(host, np.ndarray):
            host[...] = res
        else:
            host.copy_(torch.from_numpy(res))
    return bits[:B]


__all__ = ["MERGE_CUTOFF_DEFAULT", "ShuffleConfig", "ShuffleReport", "MergeRange", "merge_plan", "merge_rounds",
           "singleton_rounds", "merge_task_indices", "fisher_yates", "merge", "merge_shuffle",
           "merge_shuffle_parallel", "batched_shuffle", "advance_state"]
