"""Golden outputs of the UNMODIFIED reference's Rao-Sandelius shuffles
(splitshuffle.rs_shuffle_parallel / rs_shuffle, _kernels.rs_range_inplace),
§8 row F2.  Build container only:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_rs_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

import shufflekit as sk
from shufflekit import _kernels
from shufflekit.shufflers import ShuffleConfig
from shufflekit.splitshuffle import rs_shuffle, rs_shuffle_parallel

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    g = {"parallel": [], "sequential": [], "range": []}
    for n, cutoff, seed in [(0, None, 1), (1, None, 1), (2, None, 3), (10, 1, 4), (100, 4, 5), (1000, 16, 6),
                            (5000, None, 7), (16384, None, 8), (16385, None, 9), (40_000, None, 10),
                            (100_000, None, 11), (100_000, 1, 12), (100_000, 100_000, 13), (300_007, 1000, 14),
                            (1 << 20, None, 0), (1 << 22, None, 15), (3_000_017, 64, 16)]:
        a = np.arange(n, dtype=np.int64)
        rep = rs_shuffle_parallel(a, ShuffleConfig(cutoff=cutoff, threads=8), sk.BitSource(seed))
        c = {"n": n, "cutoff": cutoff, "seed": seed, "bits": int(rep.bits), "sha_u64": sha(a.astype("<u8")),
             "head": a[:8].tolist()}
        if n <= 1000:
            c["perm"] = a.tolist()
        g["parallel"].append(c)
    for n, cutoff, seed in [(0, None, 1), (1, None, 2), (50, 3, 3), (10_000, None, 4), (100_000, 500, 5),
                            (200_003, None, 6)]:
        a = np.arange(n, dtype=np.int64)
        src = sk.BitSource(seed)
        rep = rs_shuffle(a, ShuffleConfig(cutoff=cutoff), src)
        g["sequential"].append({"n": n, "cutoff": cutoff, "seed": seed, "bits": int(rep.bits),
                                "sha_u64": sha(a.astype("<u8")), "state_out": list(src.state_tuple())})
    for seed, pre, lo, hi, total, cutoff in [(3, 17, 5, 900, 1000, 32), (4, 100, 0, 20_000, 20_000, 4096),
                                             (5, 63, 100, 70_100, 70_500, 1000)]:
        src = sk.BitSource(seed)
        src.take(pre)
        st_in = list(src.state_tuple())
        a = np.arange(total, dtype=np.int64)
        _kernels.rs_range_inplace(a, lo, hi, cutoff, src)
        g["range"].append({"seed": seed, "pre": pre, "lo": lo, "hi": hi, "total": total, "cutoff": cutoff,
                           "state_in": st_in, "state_out": list(src.state_tuple()), "sha_u64": sha(a.astype("<u8"))})
    with open(os.path.join(OUT, "rs.json"), "w") as fh:
        json.dump(g, fh, indent=1)


if __name__ == "__main__":
    main()
