"""The oracle's BalancedShuffle restatement (n <= 32, oracle/shufflekit_oracle.c
ora_bs_small) pinned to the unmodified reference's outputs
(tests/golden/balanced.json from make_balanced_golden.py: balanced_shuffle,
balanced.py:219-245, and chi_counts("balanced"), _kernels.py:501-508)."""
import json
import os

import numpy as np

from oracle import oracle as O

G = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "balanced.json")))


def test_bs_small_matches_reference_shuffles():
    for case in G["shuffles"]:
        a = np.arange(case["n"], dtype=np.int64)
        st = np.array(case["state_in"], dtype=np.uint64)
        O.bs_small(a, st)
        assert a.tolist() == case["perm"], case["n"]
        assert [int(v) for v in st] == case["state_out"]
        assert int(st[3]) - case["state_in"][3] == case["bits"]


def test_bs_chi_counts_match_reference():
    for key, ref in G["chi"].items():
        n, trials, seed = (int(p[1:]) for p in key.split("_"))
        got = O.chi_counts("balanced", n, trials, seed, 1, threads=8)
        assert got.tolist() == ref, key
