"""The multi-limb BalancedShuffle oracle (oracle/balanced_oracle.py) against the unmodified
reference's outputs (tests/golden/balanced.json for n <= 32,
balanced_big.json for n = 33 .. 2^20): permutation, bit count, end state."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import balanced_oracle as BO

HERE = os.path.dirname(os.path.abspath(__file__))
SMALL = json.load(open(os.path.join(HERE, "golden", "balanced.json")))["shuffles"]
BIG = json.load(open(os.path.join(HERE, "golden", "balanced_big.json")))["shuffles"]


def _check(case):
    arr = list(range(case["n"]))
    bits, st = BO.balanced_shuffle(arr, case["state_in"])
    assert bits == case["bits"]
    assert list(st) == case["state_out"]
    if "perm" in case:
        assert arr == case["perm"]
    if "sha_u32" in case:
        assert hashlib.sha256(np.asarray(arr, dtype="<u4").tobytes()).hexdigest() == case["sha_u32"]


def test_oracle_small_goldens():
    for case in SMALL:
        _check(case)


@pytest.mark.parametrize("case", [c for c in BIG if c["n"] <= 20000],
                         ids=lambda c: f"n{c['n']}_s{c['state_in'][3]}_{c['state_in'][0] % 997}")
def test_oracle_big_goldens(case):
    _check(case)


def test_oracle_stream_matches_bitsource():
    # the oracle's stream restatement against the product BitSource (both
    # pinned to the reference's substream words elsewhere)
    import paper_1508_03167_b200 as sk
    src = sk.BitSource(12345)
    s = BO.Stream(src.state_tuple())
    for k in (1, 5, 64, 3, 70, 129, 7, 200):
        assert s.bits(k) == src.take(k)
    for b in (2, 3, 6, 1 << 40, (1 << 200) + 12345, 10 ** 70):
        assert s.below(b) == src.random_int(b)
    assert tuple(s.state()) == tuple(src.state_tuple())
