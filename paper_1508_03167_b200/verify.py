"""Uniformity harness (reference: pkg/src/shufflekit/verify.py:259-272, 566-626
and _kernels.chi_counts, _kernels.py:489-526).

chi_counts runs every trial on the GPU (one thread per trial, rank histogram in
shared memory); the histogram is identical to the reference's for the same
(algorithm, n, trials, seed, cutoff) -- trial t always uses substream t, so the
result does not depend on how trials are spread over threads.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .bitstream import BitSource, substream_seed
from .shufflers import MERGE_CUTOFF_DEFAULT

_CHI_ALGO_IDS = {"fy": 0, "merge": 1, "merge_parallel": 2, "balanced": 3}
CHI_ALGORITHMS = tuple(_CHI_ALGO_IDS)


def permutation_rank(perm) -> int:
    """Little-endian factorial-base rank (verify.py:259-272)."""
    r, f = 0, 1
    for k in range(1, len(perm)):
        f *= k
        pk = perm[k]
        r += f * sum(1 for j in range(k) if perm[j] < pk)
    return r


def chi_counts(algo: str, n: int, trials: int, seed: int, cutoff: int, threads: int = 1) -> np.ndarray:
    """Output-rank histogram over `trials` shuffles of the identity on n items."""
    if algo not in _CHI_ALGO_IDS:
        raise ValueError(f"algorithm {algo!r} is not on the GPU path (choose from {sorted(_CHI_ALGO_IDS)})")
    counts = np.zeros(math.factorial(n), dtype=np.int64)
    stream = None
    try:
        import torch
        if torch.cuda.is_available():
            stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    except ImportError:
        pass
    _lib.check(_lib.load().sk_chi_counts(_CHI_ALGO_IDS[algo], n, trials, seed & ((1 << 64) - 1), cutoff,
                                         counts.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), stream))
    return counts


@dataclass
class ChiSquareResult:
    algorithm: str
    n: int
    trials: int
    statistic: float
    df: int
    threshold: float
    passed: bool


def chi_square_threshold(df: int, quantile: float = 0.999) -> float:
    from scipy.stats import chi2
    return float(chi2.ppf(quantile, df))


def _default_cutoff(algorithm: str, cutoff: Optional[int]) -> int:
    if cutoff is not None:
        return cutoff
    if algorithm.startswith("merge"):
        return MERGE_CUTOFF_DEFAULT
    return 1


def chi_square_uniformity(algorithm, n: int, trials: int, seed: int, *, cutoff: Optional[int] = None,
                          threads: int = 1) -> ChiSquareResult:
    """Pearson chi-square over permutation ranks at the 0.999 quantile with n!-1
    degrees of freedom (verify.py:582-616)."""
    nf = math.factorial(n)
    if trials < 10 * nf:
        raise ValueError(f"need at least {10 * nf} trials for n={n}, got {trials}")
    name = algorithm if isinstance(algorithm, str) else getattr(algorithm, "__name__", "custom")
    if isinstance(algorithm, str):
        counts = chi_counts(algorithm, n, trials, seed, _default_cutoff(algorithm, cutoff), threads=threads)
    else:
        counts = [0] * nf
        for t in range(trials):
            src = BitSource(substream_seed(seed, t))
            arr = list(range(n))
            algorithm(arr, src)
            counts[permutation_rank(arr)] += 1
    expected = trials / nf
    stat = float(sum((int(c) - expected) ** 2 for c in counts) / expected)
    df = nf - 1
    thr = chi_square_threshold(df)
    return ChiSquareResult(name, n, trials, stat, df, thr, stat < thr)
