"""Whole-array fingerprints of the reference at the headline sizes.

Runs the UNMODIFIED reference (shufflekit.merge_shuffle_parallel,
shufflers.py:251-299) on int64 identity arrays at n = 2^30 (BASELINE config 3),
2^31 and a non-power-of-two 3*2^29+7, and records the SHA-256 of the whole
permuted array as little-endian uint32 and uint64, the bit count and the head.
Build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_big_golden.py

Output: tests/golden/big.json (a few hundred bytes).  Needs ~26 GB of RAM at
2^31; about a minute per case on 8 host threads.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

import shufflekit as sk
from shufflekit.shufflers import ShuffleConfig

OUT = os.path.dirname(os.path.abspath(__file__))
THREADS = os.cpu_count() or 1
CASES = [(1 << 30, 0), (1 << 31, 0), (3 * (1 << 29) + 7, 2)]


def sha_chunked(a: np.ndarray, dt: str) -> str:
    h = hashlib.sha256()
    step = 1 << 26
    for i in range(0, a.size, step):
        h.update(a[i:i + step].astype(dt).tobytes())
    return h.hexdigest()


def main():
    out = {"threads_used": THREADS, "cases": []}
    for n, seed in CASES:
        t0 = time.time()
        idx = np.arange(n, dtype=np.int64)
        rep = sk.merge_shuffle_parallel(idx, ShuffleConfig(threads=THREADS), sk.BitSource(seed))
        t1 = time.time()
        case = {"n": n, "cutoff": None, "seed": seed, "bits": int(rep.bits),
                "head": idx[:8].tolist(), "tail": idx[-2:].tolist(),
                "sha_u32": sha_chunked(idx, "<u4") if n <= (1 << 32) else None,
                "sha_u64": sha_chunked(idx, "<u8"), "ref_seconds": round(t1 - t0, 1)}
        out["cases"].append(case)
        print(n, seed, case["bits"], f"{t1 - t0:.1f}s", file=sys.stderr)
        del idx
    with open(os.path.join(OUT, "big.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
