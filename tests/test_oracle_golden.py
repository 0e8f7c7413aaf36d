"""Pin the CPU oracle (oracle/shufflekit_oracle.c) against the reference:
the reference's own known-answer tests (pkg/tests/test_bitstream.py:75-82,
94-104, 37-53) and golden outputs of the unmodified reference (tests/golden)."""
import numpy as np
import pytest

from golden import CHI, G, cutoff_of, sha
from oracle import oracle as O


def test_known_answer_substream_words():
    # pkg/tests/test_bitstream.py:80-81
    st = O.state_vec(O.substream_seed(42, 0), 0, 0, 0)
    assert O.take(st, 64) == 0x57E1FABA65107204
    st = O.state_vec(O.substream_seed(42, 1), 0, 0, 0)
    assert O.take(st, 64) == 0xFC991BCA1A1AA1AE


def test_substream_golden_words():
    for key, hexv in G["substream_take256"].items():
        seed, idx = (int(x) for x in key.split(":"))
        st = O.state_vec(O.substream_seed(seed, idx), 0, 0, 0)
        v = 0
        for _ in range(4):
            v = (v << 64) | O.take(st, 64)
        assert v == int(hexv, 16), key
    for key, v in G["substream_seed"].items():
        seed, idx = (int(x) for x in key.split(":"))
        assert O.substream_seed(seed, idx) == v


def test_take_sequences_and_state():
    for case in G["take_sequences"]:
        st = O.state_vec(case["seed"], 0, 0, 0)
        for k, hexv in zip(case["ks"], case["vals"]):
            v = 0
            rem = k
            while rem:
                step = min(rem, 64)
                v = (v << step) | O.take(st, step)
                rem -= step
            assert v == int(hexv, 16)
        assert [int(x) for x in st] == case["state"]


def test_fdr_draws():
    for case in G["fdr"]:
        st = O.state_vec(case["seed"], 0, 0, 0)
        draws = [O.fdr(st, b) for b in case["bounds"]]
        assert draws == case["draws"]
        assert int(st[3]) == case["bits"]
        assert [int(x) for x in st] == case["state"]


def test_fdr_contracts():
    # bound 1 -> 0 bits; bound 2 -> exactly one bit (test_bitstream.py:37-48)
    st = O.state_vec(3, 0, 0, 0)
    assert O.fdr(st, 1) == 0 and int(st[3]) == 0
    for seed in range(20):
        st = O.state_vec(seed, 0, 0, 0)
        assert O.fdr(st, 2) in (0, 1) and int(st[3]) == 1


@pytest.mark.parametrize("case", [c for c in G["merge_shuffle_parallel"] if c["n"] <= (1 << 24)],
                         ids=lambda c: f"n{c['n']}_c{c['cutoff']}_s{c['seed']}")
def test_merge_shuffle_parallel_golden(case):
    idx, bits = O.merge_shuffle_perm(case["n"], cutoff_of(case), case["seed"], threads=8)
    assert bits == case["bits"]
    if "perm" in case:
        assert idx.tolist() == case["perm"]
    assert idx[:8].tolist() == case["head"]
    assert sha(idx.astype("<u8")) == case["sha_u64"]


def test_merge_shuffle_parallel_golden_2p26():
    case = [c for c in G["merge_shuffle_parallel"] if c["n"] == (1 << 26) and c["seed"] == 0][0]
    idx, bits = O.merge_shuffle_perm(case["n"], cutoff_of(case), case["seed"], threads=8)
    assert bits == case["bits"] == 1724975486
    assert sha(idx.astype("<u4")) == case["sha_u32"]


def test_mid_stream_fy_and_merge():
    for case in G["mid_stream"]:
        st = np.array(case["state_in"], dtype=np.uint64)
        if case["op"] == "fy":
            a = np.arange(case["n"], dtype=np.int64)
            O.fy_range(a, 0, case["n"], st)
        else:
            a = np.arange(case["total"], dtype=np.int64)
            s, n1, n2 = case["s"], case["n1"], case["n2"]
            O.merge(a, s, s + n1, s + n1 + n2, st)
        assert [int(x) for x in st] == case["state_out"], case
        assert sha(a.astype("<u8")) == case["sha_u64"]


def test_sequential_merge_shuffle():
    for case in G["merge_shuffle_seq"]:
        a = np.arange(case["n"], dtype=np.int64)
        st = O.state_vec(case["seed"], 0, 0, 0)
        O.merge_shuffle_seq(a, cutoff_of(case), st)
        assert int(st[3]) == case["bits"]
        assert sha(a.astype("<u8")) == case["sha_u64"]


def test_batched_small():
    case = [c for c in G["batched"] if c["batch"] == 64][0]
    rows, bits = O.batched(case["batch"], case["len"], cutoff_of(case), case["seed"], threads=8)
    assert sha(rows.astype("<u4")) == case["sha_u32"]
    assert sha(bits.astype("<u8")) == case["sha_bits"]


def test_batched_config5():
    case = [c for c in G["batched"] if c["batch"] == 65536][0]
    rows, bits = O.batched(case["batch"], case["len"], cutoff_of(case), case["seed"], threads=8)
    assert rows[0, :8].tolist() == case["row0"] == [3134, 3888, 2523, 694, 2839, 4015, 1321, 806]
    assert int(bits[0]) == case["bits0"] == 47245
    assert sha(rows.astype("<u4")) == case["sha_u32"]


@pytest.mark.parametrize("key", sorted(CHI))
def test_chi_counts(key):
    parts = key.split("_")
    algo = "merge_parallel" if key.startswith("merge_parallel") else key.split("_")[0]
    n = 6
    for p in parts:
        if p.startswith("n") and p[1:].isdigit():
            n = int(p[1:])
    cut = int([p for p in parts if p.startswith("c") and p[1:].isdigit()][0][1:]) if any(
        p.startswith("c") and p[1:].isdigit() for p in parts) else 1
    trials = int([p for p in parts if p.startswith("t")][0][1:])
    seed = int([p for p in parts if p.startswith("s") and p[1:].isdigit()][0][1:])
    counts = O.chi_counts(algo, n, trials, seed, cut, threads=8)
    assert np.array_equal(counts, CHI[key])
