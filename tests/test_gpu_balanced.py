"""BalancedShuffle on the GPU (n <= 32 slice):
bit-exact against the reference's goldens (balanced_shuffle with state
write-back, chi_counts("balanced") histograms) and the oracle."""
import json
import os

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


def test_balanced_beyond_small_slice_refused():
    with pytest.raises(NotImplementedError):
        sk.balanced_shuffle(torch.arange(33, device="cuda"), sk.ShuffleConfig(), sk.BitSource(1))
