"""CPU check of the closed forms the CUDA kernels implement (decomp_model.py)
against the serial reference semantics, on random bit streams."""
import random

import numpy as np
import pytest

from decomp_model import (BitCursor, fy_serial, leaf_apply_model, merge_phase1_model, merge_serial,
                          spec_decode_model, stream_bits, tail_apply, tail_plan_model)
from oracle import oracle as O


@pytest.mark.parametrize("seed", range(4))
def test_leaf_chain_form(seed):
    rng = random.Random(seed)
    for _ in range(60):
        m = rng.choice([1, 2, 3, 5, 17, 100, 1000, 4096])
        draws = [0] + [rng.randint(0, i) for i in range(1, m)]
        vals = list(range(m))
        assert fy_serial(vals, draws) == leaf_apply_model(vals, draws)


def test_leaf_chain_form_on_reference_draws():
    # draws of a real leaf substream (FDR via the oracle) reproduce the oracle's FY
    m = 3000
    st = O.state_vec(O.substream_seed(123, 0), 0, 0, 0)
    draws = [0] * m
    for i in range(m - 1, 0, -1):
        draws[i] = O.fdr(st, i + 1)
    a = np.arange(m, dtype=np.int64)
    O.fy_range(a, 0, m, O.state_vec(O.substream_seed(123, 0), 0, 0, 0))
    assert leaf_apply_model(list(range(m)), draws) == a.tolist()


@pytest.mark.parametrize("seed", range(6))
def test_merge_window_and_tail_forms(seed):
    rng = random.Random(100 + seed)
    for _ in range(40):
        n1 = rng.choice([1, 2, 3, 7, 50, 333, 1000])
        n2 = rng.choice([1, 2, 3, 9, 64, 500, 1200])
        bits = stream_bits(rng.getrandbits(64), 16 * (n1 + n2) + 4000)
        vals = list(range(n1 + n2))
        out, t, aex, p1, draws, _ = merge_serial(vals, n1, n2, bits)
        mo, mt, maex = merge_phase1_model(vals, n1, n2, bits, T=rng.choice([1, 4, 16, 64]))
        assert (mt, maex) == (t, aex)
        assert mo == p1
        assert tail_apply(p1, tail_plan_model(n1 + n2, t, draws)) == out


def test_merge_model_matches_oracle_merge():
    # the serial model merge == oracle merge (reference _merge) on a real substream
    for seed, n1, n2 in ((1, 100, 120), (2, 1000, 1), (3, 1, 700), (4, 2048, 2048)):
        sseed = O.substream_seed(seed, 7)
        bits = stream_bits(sseed, 40 * (n1 + n2) + 4000)
        out, t, aex, p1, draws, used = merge_serial(list(range(n1 + n2)), n1, n2, bits)
        a = np.arange(n1 + n2, dtype=np.int64)
        st = O.state_vec(sseed, 0, 0, 0)
        O.merge(a, 0, n1, n1 + n2, st)
        assert a.tolist() == out and int(st[3]) == used


@pytest.mark.parametrize("m", [2, 3, 5, 17, 64, 100, 1000, 4097, 20000])
def test_spec_decode_form(m):
    # the batched start-offset speculation of leaf_decode_spec_kernel equals the serial FDR loop
    for seed in (0, 1):
        bits = stream_bits(O.substream_seed(seed, m), 24 * m + 4096)
        cur = BitCursor(bits)
        want = [0] * m
        for i in range(m - 1, 0, -1):
            want[i] = cur.fdr(i + 1)
        got, used, batches = spec_decode_model(m, bits)
        assert got == want and used == cur.pos
        for H, lanes in ((1, 32), (2, 8), (6, 32)):
            got, used, _ = spec_decode_model(m, bits, H=H, lanes=lanes)
            assert got == want and used == cur.pos


def test_spec_decode_form_on_oracle_draws():
    m = 3000
    st = O.state_vec(O.substream_seed(7, 3), 0, 0, 0)
    want = [0] * m
    for i in range(m - 1, 0, -1):
        want[i] = O.fdr(st, i + 1)
    bits = stream_bits(O.substream_seed(7, 3), 24 * m)
    got, _, batches = spec_decode_model(m, bits)
    assert got == want
    assert batches < m / 3     # several draws per batch
