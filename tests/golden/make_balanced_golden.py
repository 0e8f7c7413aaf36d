"""Goldens for BalancedShuffle from the UNMODIFIED
reference.  Build container only:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_balanced_golden.py

balanced.json: balanced_shuffle (balanced.py:219-245) on identity arrays of
n <= 32 from fresh and mid-stream BitSources (permutation, bits, end state),
and _kernels.chi_counts("balanced", ...) histograms (_kernels.py:501-508).
"""
import json
import os

import numpy as np

import shufflekit as sk
from shufflekit import _kernels
from shufflekit.balanced import balanced_shuffle
from shufflekit.shufflers import ShuffleConfig

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    cases = []
    for n in list(range(0, 33)) + [32, 31, 17]:
        for seed, pre in ((n * 7 + 1, 0), (n + 1000, 13), (2 ** 64 - 1 - n, 64)):
            src = sk.BitSource(seed)
            if pre:
                src.take(pre)
            st0 = [int(x) for x in src.state_tuple()]
            arr = list(range(n))
            rep = balanced_shuffle(arr, ShuffleConfig(), src)
            cases.append({"n": n, "state_in": st0, "perm": arr, "bits": int(rep.bits),
                          "state_out": [int(x) for x in src.state_tuple()]})
    chi = {}
    for n, trials, seed in ((5, 200_000, 1), (6, 1_000_000, 2), (7, 500_000, 3), (3, 10_000, 4)):
        chi[f"n{n}_t{trials}_s{seed}"] = _kernels.chi_counts("balanced", n, trials, seed, 1,
                                                             threads=os.cpu_count() or 1).tolist()
    with open(os.path.join(OUT, "balanced.json"), "w") as fh:
        json.dump({"shuffles": cases, "chi": chi}, fh)


if __name__ == "__main__":
    main()
