"""Host-side logic of the drop-in package (no GPU): schedule, BitSource state
protocol, closed-form state advance."""
import random

import numpy as np

from golden import G
from oracle import oracle as O
from paper_1508_03167_b200 import bitstream as B
from paper_1508_03167_b200 import shufflers as S


def test_bitsource_matches_reference_goldens():
    for case in G["take_sequences"]:
        src = B.BitSource(case["seed"])
        assert [hex(src.take(k)) for k in case["ks"]] == case["vals"]
        assert list(src.state_tuple()) == case["state"]
    for case in G["fdr"]:
        src = B.BitSource(case["seed"])
        assert [src.random_int(b) for b in case["bounds"]] == case["draws"]
        assert list(src.state_tuple()) == case["state"]
    assert B.BitSource(42).split_substream(0).take(64) == 0x57E1FABA65107204


def test_advance_state_closed_form():
    rng = random.Random(5)
    for _ in range(300):
        src = B.BitSource(rng.getrandbits(64))
        src.take(rng.randint(0, 200))
        st0 = src.state_tuple()
        T = rng.choice([0, 1, 5, 63, 64, 65, 127, 128, 1000, rng.randint(0, 5000)])
        left = T
        while left:
            k = min(left, 64)
            src.take(k)
            left -= k
        assert B.advance_state(st0, T) == src.state_tuple()


def test_schedule_matches_reference_formulas():
    for n, cutoff in ((0, 1), (1, 1), (6, 1), (6, 2), (100, 7), (10 ** 6, 65536), ((1 << 20) + 3, 1000)):
        c, q, bounds = S.merge_plan(n, cutoff)
        assert (n >> c) <= cutoff and (c == 0 or (n >> (c - 1)) > cutoff)
        assert bounds == [(n * i) >> c for i in range(q + 1)]
        rounds, idx = S.merge_rounds(n, cutoff), S.merge_task_indices(n, cutoff)
        assert len(rounds) == c == len(idx)
        for r, (lv, il) in enumerate(zip(rounds, idx), start=1):
            p = 1 << (r - 1)
            assert [i for _, i in il] == list(range(0, q, 2 * p))
            assert [s for s, _ in il] == [r * q + i for i in range(0, q, 2 * p)]
            assert lv == [(bounds[i], bounds[i + p], bounds[min(i + 2 * p, q)]) for i in range(0, q, 2 * p)]


def test_config_validation():
    import pytest
    with pytest.raises(ValueError):
        S.ShuffleConfig(cutoff=0)
    with pytest.raises(ValueError):
        S.ShuffleConfig(threads=0)
    with pytest.raises(ValueError):
        S.MergeRange(-1, 1, 1)
    with pytest.raises(ValueError):
        B.BitSource(1).random_int(0)
    with pytest.raises(ValueError):
        B.substream_seed(1, -1)


def test_oracle_tasked_equals_sequential_pure_python_schedule():
    # the frozen schedule == leaf/merge tasks on substreams, run on the oracle
    n, cutoff, seed = 5000, 300, 11
    a = np.arange(n, dtype=np.int64)
    bits = O.merge_shuffle_tasked(a, cutoff, seed)
    b = np.arange(n, dtype=np.int64)
    c, q, bounds = S.merge_plan(n, cutoff)
    tot = 0
    for i in range(q):
        st = O.state_vec(O.substream_seed(seed, i), 0, 0, 0)
        O.fy_range(b, bounds[i], bounds[i + 1], st)
        tot += int(st[3])
    for lv, il in zip(S.merge_rounds(n, cutoff), S.merge_task_indices(n, cutoff)):
        for (j, k, l), (sidx, _) in zip(lv, il):
            st = O.state_vec(O.substream_seed(seed, sidx), 0, 0, 0)
            O.merge(b, j, k, l, st)
            tot += int(st[3])
    assert np.array_equal(a, b) and bits == tot


def test_tail_length_statistics_behind_the_capacity_bound():
    # csrc/engine.cu tail_capacity sizes a round's tail buffers as
    # sum 0.80 sqrt(N) + 9 sqrt(sum 0.37 N): the tail of a pair of N elements
    # has L = N - t insertions, t = min(select0(n1), select1(n2)) on its bit
    # stream (_kernels.py:104-121).  Check the constants on pair streams.
    rng = np.random.default_rng(3)
    for N in (1 << 10, 1 << 14):
        n1 = N // 2
        L = []
        for _ in range(3000):
            b = rng.integers(0, 2, 2 * N + 10)
            tz = np.searchsorted(np.cumsum(1 - b), n1 + 1)
            to = np.searchsorted(np.cumsum(b), N - n1 + 1)
            L.append(N - min(tz, to))
        L = np.asarray(L, dtype=np.float64)
        assert abs(L.mean() / np.sqrt(N) - 0.80) < 0.04
        assert abs(L.var() / N - 0.37) < 0.05
        assert L.max() < 0.80 * np.sqrt(N) + 9 * np.sqrt(0.37 * N)
