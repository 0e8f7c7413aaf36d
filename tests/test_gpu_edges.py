"""Edge cases on the GPU against the oracle: sizes around powers of two,
extreme cutoffs (leaves above 65536 take the serial leaf path), odd batch
shapes, long single-stream Fisher-Yates, and the splitting shuffle with a
huge cutoff."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1508_03167_b200 as sk  # noqa: E402
from paper_1508_03167_b200 import splitshuffle as S  # noqa: E402
from oracle import oracle as O  # noqa: E402


def run(n, cutoff, seed, dt):
    x = torch.arange(n, dtype=dt, device="cuda")
    rep = sk.merge_shuffle_parallel(x, sk.ShuffleConfig(cutoff=cutoff), sk.BitSource(seed))
    ref, bits = O.merge_shuffle_perm(n, cutoff if cutoff else 65536, seed)
    assert rep.bits == bits
    assert np.array_equal(x.cpu().numpy().astype(np.int64), ref)


@pytest.mark.parametrize("k", [16, 17, 20])
@pytest.mark.parametrize("d", [-1, 0, 1])
@pytest.mark.parametrize("dt", [torch.int32, torch.int64])
def test_sizes_around_powers_of_two(k, d, dt):
    run((1 << k) + d, None, 1000 + k + d, dt)


@pytest.mark.parametrize("cutoff", [2, 3, 5, 65535, 65537, 100_000, 1 << 20])
def test_extreme_cutoffs(cutoff):
    run(300_001, cutoff, cutoff, torch.int32)


def test_batched_odd_shapes():
    # (2049..4096 / 4097..8192-element pure Fisher-Yates leaves: the small v3
    # kernels in place; odd lengths: unaligned array starts)
    for B, L, cutoff in [(3, 100_003, 1000), (7, 65_537, None), (1000, 1, None), (5, 2, 1),
                         (333, 3001, None), (129, 4096, None), (65, 5003, None), (17, 8192, None),
                         (9, 20_001, 2500)]:
        x = torch.arange(L, dtype=torch.int64, device="cuda").repeat(B, 1).contiguous()
        bits = sk.batched_shuffle(x, sk.ShuffleConfig(cutoff=cutoff), 77)
        ref, rbits = O.batched(B, L, cutoff if cutoff else 65536, 77)
        assert np.array_equal(bits.astype(np.int64), rbits.astype(np.int64))
        assert np.array_equal(x.cpu().numpy(), ref)


@pytest.mark.parametrize("m", [65_535, 65_536, 65_537, 300_000])
def test_long_fisher_yates(m):
    x = torch.arange(m, dtype=torch.int32, device="cuda")
    src = sk.BitSource(5)
    src.take(13)
    st = np.array(src.state_tuple(), dtype=np.uint64)
    sk.fisher_yates(x, src)
    a = np.arange(m, dtype=np.int64)
    O.fy_range(a, 0, m, st)
    assert np.array_equal(x.cpu().numpy(), a)
    assert list(src.state_tuple()) == [int(v) for v in st]


def test_rs_sequential_huge_cutoff():
    # leaves above 65536 elements take the serial leaf kernel
    n = 200_000
    x = torch.arange(n, dtype=torch.int64, device="cuda")
    src = sk.BitSource(9)
    S.rs_shuffle(x, sk.ShuffleConfig(cutoff=150_000), src)
    a = np.arange(n, dtype=np.int64)
    st = O.state_vec(9, 0, 0, 0)
    O.rs_range(a, 0, n, 150_000, st)
    assert np.array_equal(x.cpu().numpy(), a)
    assert list(src.state_tuple()) == [int(v) for v in st]


def test_python_sequences_of_any_items():
    # lists of floats, strings, bools, huge ints and objects are reordered as
    # items (index permutation on the GPU), never coerced to int64
    n, cutoff, seed = 5000, 64, 11
    ref, bits = O.merge_shuffle_perm(n, cutoff, seed)
    for items in ([i + 0.5 for i in range(n)], [f"s{i}" for i in range(n)], [bool(i & 1) for i in range(n)],
                  [2 ** 70 + i for i in range(n)], [(i, None) for i in range(n)]):
        lst = list(items)
        rep = sk.merge_shuffle_parallel(lst, sk.ShuffleConfig(cutoff=cutoff), sk.BitSource(seed))
        assert rep.bits == bits
        assert lst == [items[i] for i in ref]
    lst = [f"t{i}" for i in range(100)]
    src = sk.BitSource(3)
    st = O.state_vec(3, 0, 0, 0)
    sk.fisher_yates(lst, src)
    a = np.arange(100, dtype=np.int64)
    O.fy_range(a, 0, 100, st)
    assert lst == [f"t{i}" for i in a]


def test_tensor_on_its_own_device_and_stream():
    # a tensor is shuffled on the current stream of ITS device
    x = torch.arange(100_000, dtype=torch.int32, device="cuda:0")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        sk.merge_shuffle_parallel(x, sk.ShuffleConfig(cutoff=1000), sk.BitSource(4))
    s.synchronize()
    ref, _ = O.merge_shuffle_perm(100_000, 1000, 4)
    assert np.array_equal(x.cpu().numpy(), ref.astype(np.int32))


@pytest.mark.parametrize("n,cutoff,dt", [(1 << 20, None, torch.int32), (3_000_001, None, torch.int64),
                                         (300_007, 4096, torch.int32), (70_000, 65536, torch.int32),
                                         (5000, 1000, torch.int32), (9, 2, torch.int32)])
def test_both_leaf_decodes(n, cutoff, dt):
    # the warp-per-leaf speculative decode (jobs of few leaves) and the lane-per-leaf decode
    # produce the same draws: same permutation, same bit count, both equal to the oracle's
    import ctypes
    from paper_1508_03167_b200 import _lib
    lib = _lib.load()
    lib.sk_debug_set.argtypes = [ctypes.c_int, ctypes.c_int]
    try:
        for spec_max in (0, 1 << 30):
            assert lib.sk_debug_set(8, spec_max) == 0
            run(n, cutoff, 4242, dt)
    finally:
        lib.sk_debug_set(8, 1024)


def test_speculative_decode_mid_stream():
    # one long Fisher-Yates on a stream entered mid-word (prefix bits) through the warp-per-leaf decode
    for m in (2, 3, 64, 65, 4097, 65_536):
        x = torch.arange(m, dtype=torch.int32, device="cuda")
        src = sk.BitSource(9)
        src.take(29)
        st = np.array(src.state_tuple(), dtype=np.uint64)
        sk.fisher_yates(x, src)
        a = np.arange(m, dtype=np.int64)
        O.fy_range(a, 0, m, st)
        assert np.array_equal(x.cpu().numpy().astype(np.int64), a)
        assert tuple(int(v) for v in st) == tuple(src.state_tuple())
