"""BalancedShuffle on the GPU: bit-exact against
the reference's goldens (balanced_shuffle with state write-back for n <= 32
and for n = 33 .. 2^20, chi_counts("balanced") histograms) and the oracles
(the C restatement for n <= 32, oracle/balanced_oracle.py beyond)."""
import hashlib
import json
import os
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1508_03167_b200 as sk  # noqa: E402
from paper_1508_03167_b200 import verify as V  # noqa: E402
from oracle import oracle as O  # noqa: E402

G = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "balanced.json")))
BIG = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "balanced_big.json")))["shuffles"]


@pytest.mark.parametrize("dtype", [torch.int32, torch.int64, "list"])
def test_balanced_shuffle_reference_goldens(dtype):
    for case in G["shuffles"]:
        src = sk.BitSource(0)
        src.set_state_tuple(case["state_in"])
        if dtype == "list":
            x = [f"e{i}" for i in range(case["n"])]
            rep = sk.balanced_shuffle(x, sk.ShuffleConfig(), src)
            got = [int(s[1:]) for s in x]
        else:
            x = torch.arange(case["n"], dtype=dtype, device="cuda")
            rep = sk.balanced_shuffle(x, sk.ShuffleConfig(), src)
            got = x.cpu().tolist()
        assert got == case["perm"], case["n"]
        assert rep.bits == case["bits"] and list(src.state_tuple()) == case["state_out"]


def test_balanced_chi_counts_reference():
    for key, ref in G["chi"].items():
        n, trials, seed = (int(p[1:]) for p in key.split("_"))
        assert V.chi_counts("balanced", n, trials, seed, 1).tolist() == ref, key


def test_balanced_random_states_against_oracle():
    rng = np.random.default_rng(17)
    for _ in range(200):
        n = int(rng.integers(0, 33))
        src = sk.BitSource(int(rng.integers(0, 2 ** 63)))
        src.take(int(rng.integers(0, 130)))
        st = np.array(src.state_tuple(), dtype=np.uint64)
        a = np.arange(n, dtype=np.int64)
        O.bs_small(a, st)
        x = torch.arange(n, dtype=torch.int64, device="cuda")
        sk.balanced_shuffle(x, sk.ShuffleConfig(), src)
        assert np.array_equal(x.cpu().numpy(), a)
        assert list(src.state_tuple()) == [int(v) for v in st]


def test_balanced_chi_square_passes():
    r = V.chi_square_uniformity("balanced", 6, 1_000_000, 5)
    assert r.passed


@pytest.mark.parametrize("case", BIG, ids=lambda c: f"n{c['n']}_{c['state_in'][3]}_{c['state_in'][0] % 997}")
def test_balanced_multilimb_reference_goldens(case):
    # n = 33 .. 2^20: multi-limb class sizes, dice rolls and unranking
    dtype = torch.int32 if case["n"] % 2 else torch.int64
    src = sk.BitSource(0)
    src.set_state_tuple(case["state_in"])
    x = torch.arange(case["n"], dtype=dtype, device="cuda")
    t0 = time.perf_counter()
    rep = sk.balanced_shuffle(x, sk.ShuffleConfig(), src)
    dt = time.perf_counter() - t0
    a = x.cpu().numpy()
    assert rep.bits == case["bits"] and list(src.state_tuple()) == case["state_out"]
    assert a[:8].tolist() == case["head"]
    assert hashlib.sha256(a.astype("<u4").tobytes()).hexdigest() == case["sha_u32"]
    if "perm" in case:
        assert a.tolist() == case["perm"]
    print(f"balanced n={case['n']}: {dt * 1e3:.1f} ms")


def test_balanced_multilimb_random_states_against_oracle():
    from oracle import balanced_oracle as BO
    rng = np.random.default_rng(29)
    for _ in range(60):
        n = int(rng.integers(33, 3000))
        src = sk.BitSource(int(rng.integers(0, 2 ** 63)))
        src.take(int(rng.integers(0, 200)))
        ref = list(range(n))
        bits, st = BO.balanced_shuffle(ref, src.state_tuple())
        x = torch.arange(n, dtype=torch.int64, device="cuda")
        rep = sk.balanced_shuffle(x, sk.ShuffleConfig(), src)
        assert x.cpu().tolist() == ref, n
        assert rep.bits == bits and tuple(src.state_tuple()) == tuple(st)


def test_balanced_items_list_multilimb():
    from oracle import balanced_oracle as BO
    src = sk.BitSource(77)
    items = [f"v{i}" for i in range(500)]
    ref = list(items)
    BO.balanced_shuffle(ref, src.state_tuple())
    sk.balanced_shuffle(items, sk.ShuffleConfig(), src)
    assert items == ref


def test_balanced_beyond_supported_refused():
    with pytest.raises(NotImplementedError):
        sk.balanced_shuffle(torch.arange((1 << 20) + 1, device="cuda"), sk.ShuffleConfig(), sk.BitSource(1))
