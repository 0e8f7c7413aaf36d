"""F2 oracle pin: the C restatement of the Rao-Sandelius shuffles against the
reference's own outputs (tests/golden/rs.json, make_rs_golden.py)."""
import numpy as np
import pytest

from golden import RS, sha
from oracle import oracle as O


def cut(c):
    return 4096 if c["cutoff"] is None else c["cutoff"]  # RS_CUTOFF_DEFAULT (splitshuffle.py:27)


@pytest.mark.parametrize("case", RS["parallel"], ids=lambda c: f"n{c['n']}_c{c['cutoff']}_s{c['seed']}")
def test_rs_parallel(case):
    a = np.arange(case["n"], dtype=np.int64)
    bits = O.rs_parallel(a, cut(case), case["seed"])
    assert bits == case["bits"]
    assert sha(a.astype("<u8")) == case["sha_u64"]
    if "perm" in case:
        assert a.tolist() == case["perm"]


@pytest.mark.parametrize("case", RS["sequential"], ids=lambda c: f"n{c['n']}_s{c['seed']}")
def test_rs_sequential(case):
    a = np.arange(case["n"], dtype=np.int64)
    st = O.state_vec(case["seed"], 0, 0, 0)
    O.rs_range(a, 0, case["n"], cut(case), st)
    assert int(st[3]) == case["bits"]
    assert [int(x) for x in st] == case["state_out"]
    assert sha(a.astype("<u8")) == case["sha_u64"]


@pytest.mark.parametrize("case", RS["range"], ids=lambda c: f"s{c['seed']}")
def test_rs_range_mid_stream(case):
    a = np.arange(case["total"], dtype=np.int64)
    st = np.array(case["state_in"], dtype=np.uint64)
    O.rs_range(a, case["lo"], case["hi"], case["cutoff"], st)
    assert [int(x) for x in st] == case["state_out"]
    assert sha(a.astype("<u8")) == case["sha_u64"]
