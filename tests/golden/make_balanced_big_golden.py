"""Goldens for BalancedShuffle beyond the machine-word slice (SURVEY.md
section 8 row F1, n = 33 .. 2^20) from the UNMODIFIED reference.  Build
container only (the reference's pure-Python big-integer path; ~4 min with 2^18..2^20):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_balanced_big_golden.py

balanced_big.json: balanced_shuffle (balanced.py:219-245) on identity arrays
from fresh and mid-stream BitSources: bits, end state, the SHA-256 of the
permutation as little-endian uint32, its head, and the whole permutation for
n <= 600.
"""
import hashlib
import json
import os

import numpy as np

import shufflekit as sk
from shufflekit.balanced import balanced_shuffle
from shufflekit.shufflers import ShuffleConfig

OUT = os.path.dirname(os.path.abspath(__file__))
SIZES = [33, 34, 40, 47, 63, 64, 65, 96, 100, 127, 128, 129, 200, 255, 256, 257, 333, 500, 511, 512, 513, 600,
         1000, 1023, 1024, 1025, 2047, 2048, 3000, 4093, 4096, 5000, 8191, 10007, 16384, 30000, 65535, 65536,
         100000, 131072, 1 << 18, 1 << 19, 1 << 20]


def main():
    cases = []
    for n in SIZES:
        pres = ((0,), (13,), (64, 5)) if n <= 4096 else (((0,), (37,)) if n <= 131072 else ((0,),))
        for q, pre in enumerate(pres):
            src = sk.BitSource((n * 2654435761 + 17 * q) % (1 << 64))
            for k in pre:
                if k:
                    src.take(k)
            st0 = [int(x) for x in src.state_tuple()]
            arr = list(range(n))
            rep = balanced_shuffle(arr, ShuffleConfig(), src)
            a = np.asarray(arr, dtype="<u4")
            case = {"n": n, "state_in": st0, "bits": int(rep.bits), "state_out": [int(x) for x in src.state_tuple()],
                    "sha_u32": hashlib.sha256(a.tobytes()).hexdigest(), "head": arr[:8]}
            if n <= 600:
                case["perm"] = arr
            cases.append(case)
            print(n, pre, rep.bits, flush=True)
    with open(os.path.join(OUT, "balanced_big.json"), "w") as fh:
        json.dump({"shuffles": cases}, fh)


if __name__ == "__main__":
    main()
