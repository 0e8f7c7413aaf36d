"""F2 on the GPU: the Rao-Sandelius shuffles through the C ABI against the
reference's own outputs (tests/golden/rs.json) and the pinned oracle."""
import numpy as np
import pytest

from golden import RS, sha

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1508_03167_b200 as sk  # noqa: E402
from paper_1508_03167_b200 import splitshuffle as S  # noqa: E402
from oracle import oracle as O  # noqa: E402


@pytest.mark.parametrize("case", RS["parallel"], ids=lambda c: f"n{c['n']}_c{c['cutoff']}_s{c['seed']}")
@pytest.mark.parametrize("dtype", [torch.int32, torch.int64])
def test_rs_parallel_golden(case, dtype):
    x = torch.arange(case["n"], dtype=dtype, device="cuda")
    rep = S.rs_shuffle_parallel(x, sk.ShuffleConfig(cutoff=case["cutoff"], threads=8), sk.BitSource(case["seed"]))
    assert rep.bits == case["bits"]
    a = x.cpu().numpy().astype(np.int64)
    assert sha(a.astype("<u8")) == case["sha_u64"]
    if "perm" in case:
        assert a.tolist() == case["perm"]


@pytest.mark.parametrize("case", RS["sequential"], ids=lambda c: f"n{c['n']}_s{c['seed']}")
def test_rs_sequential_golden(case):
    x = torch.arange(case["n"], dtype=torch.int64, device="cuda")
    src = sk.BitSource(case["seed"])
    rep = S.rs_shuffle(x, sk.ShuffleConfig(cutoff=case["cutoff"]), src)
    assert rep.bits == case["bits"]
    assert list(src.state_tuple()) == case["state_out"]
    assert sha(x.cpu().numpy().astype("<u8")) == case["sha_u64"]


@pytest.mark.parametrize("case", RS["range"], ids=lambda c: f"s{c['seed']}")
def test_rs_range_mid_stream_golden(case):
    x = torch.arange(case["total"], dtype=torch.int64, device="cuda")
    src = sk.BitSource(0)
    src.set_state_tuple(case["state_in"])
    S.rs_range(x, case["lo"], case["hi"], case["cutoff"], src)
    assert list(src.state_tuple()) == case["state_out"]
    assert sha(x.cpu().numpy().astype("<u8")) == case["sha_u64"]


def test_rs_parallel_random_against_oracle():
    rng = np.random.default_rng(41)
    for _ in range(10):
        n = int(rng.integers(0, 400_000))
        cutoff = int(rng.choice([1, 3, 100, 4096, 20_000]))
        seed = int(rng.integers(0, 2 ** 63))
        a = np.arange(n, dtype=np.int64)
        bits = O.rs_parallel(a, cutoff, seed)
        x = torch.arange(n, dtype=torch.int32, device="cuda")
        rep = S.rs_shuffle_parallel(x, sk.ShuffleConfig(cutoff=cutoff), sk.BitSource(seed))
        assert rep.bits == bits
        assert np.array_equal(x.cpu().numpy(), a.astype(np.int32))


def test_rs_parallel_2p26_validity():
    n = 1 << 26
    x = torch.arange(n, dtype=torch.int32, device="cuda")
    rep = S.rs_shuffle_parallel(x, sk.ShuffleConfig(), sk.BitSource(5))
    a = np.arange(n, dtype=np.int64)
    bits = O.rs_parallel(a, 4096, 5)
    assert rep.bits == bits
    assert np.array_equal(x.cpu().numpy(), a.astype(np.int32))
