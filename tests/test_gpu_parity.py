"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
outputs and the CPU oracle, bit-exact (integer/permutation work: no tolerance)."""
import numpy as np
import pytest

from golden import CHI, CHI_STATS, G, cutoff_of, sha

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1508_03167_b200 as sk  # noqa: E402
from oracle import oracle as O  # noqa: E402


def gpu_perm(n, cutoff, seed, dtype=torch.int64):
    x = torch.arange(n, dtype=dtype, device="cuda")
    rep = sk.merge_shuffle_parallel(x, sk.ShuffleConfig(cutoff=cutoff), sk.BitSource(seed))
    torch.cuda.synchronize()
    return x, rep


SMALL = [c for c in G["merge_shuffle_parallel"] if c["n"] <= 100_000]
BIG = [c for c in G["merge_shuffle_parallel"] if c["n"] > 100_000]


@pytest.mark.parametrize("case", SMALL, ids=lambda c: f"n{c['n']}_c{c['cutoff']}_s{c['seed']}")
@pytest.mark.parametrize("dtype", [torch.int32, torch.int64])
def test_merge_shuffle_parallel_small(case, dtype):
    x, rep = gpu_perm(case["n"], case["cutoff"], case["seed"], dtype)
    assert rep.bits == case["bits"]
    a = x.cpu().numpy().astype(np.int64)
    if "perm" in case:
        assert a.tolist() == case["perm"]
    assert sha(a.astype("<u8")) == case["sha_u64"]


@pytest.mark.parametrize("case", BIG, ids=lambda c: f"n{c['n']}_c{c['cutoff']}_s{c['seed']}")
def test_merge_shuffle_parallel_big(case):
    x, rep = gpu_perm(case["n"], case["cutoff"], case["seed"], torch.int32)
    assert rep.bits == case["bits"]
    a = x.cpu().numpy()
    assert a[:8].tolist() == case["head"]
    assert sha(a.astype("<u4")) == case["sha_u32"]


def test_config1_identity_2p20_bits_and_head():
    # BASELINE config 1 / SURVEY Appendix B
    x, rep = gpu_perm(1 << 20, None, 0, torch.int32)
    a = x.cpu().numpy()
    assert rep.bits == 20642558
    assert a[:8].tolist() == [31015, 50941, 611601, 90548, 556729, 372014, 358856, 1037783]
    assert a[-2:].tolist() == [336614, 950641]
    assert sha(a.astype("<u4")) == "6925255c4af1bba6db58298875f584606717738eed42ca81674550e28698b8a9"


def test_config2_payload_2p26_against_oracle():
    n = 1 << 26
    rng = np.random.default_rng(2026)
    payload = rng.integers(0, 2 ** 32, n, dtype=np.uint32)
    idx, bits = O.merge_shuffle_perm(n, 65536, 0, threads=8)
    expect = payload[idx]
    x = torch.from_numpy(payload.view(np.int32)).cuda()
    rep = sk.merge_shuffle_parallel(x, sk.ShuffleConfig(), sk.BitSource(0))
    assert rep.bits == bits == 1724975486
    assert np.array_equal(x.cpu().numpy().view(np.uint32), expect)


def test_numpy_host_path_and_payload_types():
    n = 200_003
    idx, bits = O.merge_shuffle_perm(n, 4096, 77)
    for dt in (np.uint32, np.int64, np.float32, np.float64):
        payload = (np.arange(n) * 3 + 1).astype(dt)
        a = payload.copy()
        rep = sk.merge_shuffle_parallel(a, sk.ShuffleConfig(cutoff=4096), sk.BitSource(77))
        assert rep.bits == bits
        assert np.array_equal(a, payload[idx])
    # 2-byte payload: index permutation on the GPU, gather on the host
    p16 = (np.arange(n) % 60000).astype(np.uint16)
    a16 = p16.copy()
    sk.merge_shuffle_parallel(a16, sk.ShuffleConfig(cutoff=4096), sk.BitSource(77))
    assert np.array_equal(a16, p16[idx])
    lst = list(range(1000))
    sk.merge_shuffle_parallel(lst, sk.ShuffleConfig(cutoff=7), sk.BitSource(3))
    ref, _ = O.merge_shuffle_perm(1000, 7, 3)
    assert lst == ref.tolist()


def test_mid_stream_entry_points():
    for case in G["mid_stream"]:
        src = sk.BitSource(0)
        src.set_state_tuple(case["state_in"])
        if case["op"] == "fy":
            x = torch.arange(case["n"], dtype=torch.int64, device="cuda")
            sk.fisher_yates(x, src)
        else:
            x = torch.arange(case["total"], dtype=torch.int64, device="cuda")
            sk.merge(x, sk.MergeRange(case["s"], case["n1"], case["n2"]), src)
        assert list(src.state_tuple()) == case["state_out"], case
        assert sha(x.cpu().numpy().astype("<u8")) == case["sha_u64"], case


def test_mid_stream_random_against_oracle():
    rng = np.random.default_rng(9)
    for _ in range(30):
        pre = int(rng.integers(0, 300))
        seed = int(rng.integers(0, 2 ** 63))
        n1, n2 = int(rng.integers(0, 3000)), int(rng.integers(0, 3000))
        s = int(rng.integers(0, 50))
        tot = s + n1 + n2 + int(rng.integers(0, 50))
        src = sk.BitSource(seed)
        src.take(pre)
        st = np.array(src.state_tuple(), dtype=np.uint64)
        a = np.arange(tot, dtype=np.int64)
        O.merge(a, s, s + n1, s + n1 + n2, st)
        x = torch.arange(tot, dtype=torch.int32, device="cuda")
        sk.merge(x, sk.MergeRange(s, n1, n2), src)
        assert np.array_equal(x.cpu().numpy(), a)
        assert list(src.state_tuple()) == [int(v) for v in st]
        m = int(rng.integers(0, 5000))
        st = np.array(src.state_tuple(), dtype=np.uint64)
        b = np.arange(m, dtype=np.int64)
        O.fy_range(b, 0, m, st)
        y = torch.arange(m, dtype=torch.int64, device="cuda")
        sk.fisher_yates(y, src)
        assert np.array_equal(y.cpu().numpy(), b)
        assert list(src.state_tuple()) == [int(v) for v in st]


def test_sequential_merge_shuffle():
    for case in G["merge_shuffle_seq"]:
        if case["n"] > 200_000:
            continue
        x = torch.arange(case["n"], dtype=torch.int64, device="cuda")
        rep = sk.merge_shuffle(x, sk.ShuffleConfig(cutoff=case["cutoff"]), sk.BitSource(case["seed"]))
        assert rep.bits == case["bits"]
        assert sha(x.cpu().numpy().astype("<u8")) == case["sha_u64"]


@pytest.mark.parametrize("which", [64, 65536])
def test_batched(which):
    case = [c for c in G["batched"] if c["batch"] == which][0]
    B, L = case["batch"], case["len"]
    x = torch.arange(L, dtype=torch.int32, device="cuda").repeat(B, 1).contiguous()
    bits = sk.batched_shuffle(x, sk.ShuffleConfig(cutoff=case["cutoff"]), case["seed"])
    a = x.cpu().numpy()
    assert a[0, :8].tolist() == case["row0"] and a[-1, :8].tolist() == case["row_last"]
    assert int(bits[0]) == case["bits0"] and int(bits.sum()) == case["bits_sum"]
    assert sha(a.astype("<u4")) == case["sha_u32"]
    assert sha(bits.astype("<u8")) == case["sha_bits"]


@pytest.mark.parametrize("key", sorted(CHI))
def test_chi_counts_equal_reference(key):
    parts = key.split("_")
    algo = "merge_parallel" if key.startswith("merge_parallel") else parts[0]
    n = next((int(p[1:]) for p in parts if p.startswith("n") and p[1:].isdigit()), 6)
    cut = next((int(p[1:]) for p in parts if p.startswith("c") and p[1:].isdigit()), 1)
    trials = next(int(p[1:]) for p in parts if p.startswith("t"))
    seed = next(int(p[1:]) for p in parts if p.startswith("s") and p[1:].isdigit())
    counts = sk.chi_counts(algo, n, trials, seed, cut)
    assert np.array_equal(counts, CHI[key])


def test_chi_square_statistic_config2():
    for cut in (65536, 1):
        r = sk.chi_square_uniformity("merge_parallel", 6, 10_000_000, 0, cutoff=cut)
        assert r.passed
        assert abs(r.statistic - CHI_STATS[str(cut)]["statistic"]) < 1e-6


def test_full_size_2p30_validity_and_bits():
    # n = 2^30 (config 3, 1 GPU): reference bits 31908987766 and head;
    # permutation validity on the whole array.
    n = 1 << 30
    x = torch.arange(n, dtype=torch.int32, device="cuda")
    rep = sk.merge_shuffle_parallel(x, sk.ShuffleConfig(), sk.BitSource(0))
    assert rep.bits == 31908987766
    assert x[:8].cpu().tolist() == [689509142, 560979983, 717555468, 1025498733, 1056958978, 1072831348,
                                    937792008, 1008664118]
    seen = torch.zeros(n // 32, dtype=torch.int32, device="cuda")
    # validity: every value exactly once (bitmap via scatter of sorted chunks)
    s, _ = torch.sort(x)
    assert torch.equal(s, torch.arange(n, dtype=torch.int32, device="cuda"))
    del s, seen


def test_full_size_2p30_host_entry_equals_device_path():
    # the pipelined host entry (chunked H2D, per-chunk leaves and local rounds
    # on two streams, top rounds, D2H) at n = 2^30: same bits and the same
    # permutation as the device-resident path
    n = 1 << 30
    x = torch.arange(n, dtype=torch.int32, device="cuda")
    rep = sk.merge_shuffle_parallel(x, sk.ShuffleConfig(), sk.BitSource(0))
    host = torch.arange(n, dtype=torch.int32).pin_memory()
    import ctypes
    from paper_1508_03167_b200 import _lib
    bits = ctypes.c_uint64(0)
    _lib.check(_lib.load().sk_merge_shuffle_parallel_host(ctypes.c_void_p(host.data_ptr()), 4, n, 65536, 0,
                                                          ctypes.byref(bits),
                                                          ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    assert bits.value == rep.bits == 31908987766
    assert torch.equal(host.to("cuda"), x)


def test_determinism_and_seed_sensitivity():
    a, _ = gpu_perm(300_000, 1000, 5, torch.int32)
    b, _ = gpu_perm(300_000, 1000, 5, torch.int32)
    c, _ = gpu_perm(300_000, 1000, 6, torch.int32)
    assert torch.equal(a, b) and not torch.equal(a, c)


@pytest.mark.parametrize("n", [1 << 20, (1 << 20) + 12345])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_peer_exchange_on_one_gpu(world, n):
    # the fused peer-memory merge of the spanning rounds (sk_merge_range_peers,
    # every part's phase 1 in turn, then the tail), parts = slices of one
    # buffer: 16-byte aligned part boundaries (TMA path) and ragged ones
    from paper_1508_03167_b200 import distributed as D
    cutoff, seed = 32768, 23
    data = torch.arange(n, dtype=torch.int32, device="cuda")
    bits = D.simulate_sharded(data, n, cutoff, seed, world, exchange="peer")
    ref, rbits = O.merge_shuffle_perm(n, cutoff, seed)
    assert bits == rbits
    assert np.array_equal(data.cpu().numpy(), ref.astype(np.int32))


def test_merge_range_peers_random_splits():
    from paper_1508_03167_b200 import distributed as D
    eng = D.CudaEngine()
    rng = np.random.default_rng(31)
    for trial in range(12):
        n1, n2 = int(rng.integers(1, 200_000)), int(rng.integers(1, 200_000))
        N = n1 + n2
        nparts = int(rng.integers(1, 9))
        cuts = sorted(int(x) for x in rng.integers(0, N, nparts - 1))
        starts = [0] + cuts + [N]
        dt = torch.int64 if trial % 2 else torch.int32
        # each part in its own buffer, at an odd element offset for some
        bufs, bases = [], []
        for k in range(nparts):
            pad = int(rng.integers(0, 3))
            b = torch.empty(starts[k + 1] - starts[k] + pad, dtype=dt, device="cuda")
            b[pad:] = torch.arange(starts[k], starts[k + 1], dtype=dt, device="cuda")
            bufs.append((b, pad))
            bases.append(b.data_ptr() + pad * b.element_size())
        seed = int(rng.integers(0, 2 ** 63))
        for k in range(nparts):
            eng.merge_peers(bases, starts, k, bufs[0][0].element_size(), n1, n2, seed, 1)
        bits = eng.merge_peers(bases, starts, 0, bufs[0][0].element_size(), n1, n2, seed, 2)
        got = torch.cat([b[pad:] for b, pad in bufs]).cpu().numpy().astype(np.int64)
        ref = np.arange(N, dtype=np.int64)
        st = O.state_vec(seed, 0, 0, 0)
        O.merge(ref, 0, n1, N, st)
        assert bits == int(st[3])
        assert np.array_equal(got, ref)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_schedule_on_one_gpu(world):
    # the multi-GPU schedule (per-shard C-ABI calls + spanning-round merges),
    # executed shard by shard on one device, equals the single-GPU result
    from paper_1508_03167_b200 import distributed as D
    n, cutoff, seed = (1 << 20) + 12345, 32768, 17
    data = torch.arange(n, dtype=torch.int32, device="cuda")
    bits = D.simulate_sharded(data, n, cutoff, seed, world)
    ref, rbits = O.merge_shuffle_perm(n, cutoff, seed)
    assert bits == rbits
    assert np.array_equal(data.cpu().numpy(), ref.astype(np.int32))


def test_config4_sharded_2p24_uint64_golden():
    # BASELINE config 4: 8-way sharded code path, bit-exact on a 2^24 run
    from paper_1508_03167_b200 import distributed as D
    case = [c for c in G["merge_shuffle_parallel"] if c["n"] == (1 << 24)][0]
    data = torch.arange(1 << 24, dtype=torch.int64, device="cuda")
    bits = D.simulate_sharded(data, 1 << 24, None, case["seed"], 8)
    assert bits == case["bits"]
    assert sha(data.cpu().numpy().astype("<u8")) == case["sha_u64"]


def test_merge_fallback_path():
    # the tree merge's window-by-window path (taken when a tile's windows do
    # not fit shared memory or its chain is deeper than the stored starts),
    # forced for every tile: same results
    import ctypes
    from paper_1508_03167_b200 import _lib
    lib = _lib.load()
    lib.sk_debug_set.argtypes = [ctypes.c_int, ctypes.c_int]
    key, on, off = 4, 1, 0
    lib.sk_debug_set(key, on)
    try:
        for n, cutoff, seed in [(1 << 20, 65536, 0), (300_007, 4096, 1234), (100_000, 1000, 9), (5000, 7, 3)]:
            x, rep = gpu_perm(n, cutoff, seed, torch.int32)
            ref, rbits = O.merge_shuffle_perm(n, cutoff, seed)
            assert rep.bits == rbits
            assert np.array_equal(x.cpu().numpy(), ref.astype(np.int32))
        for dt in (torch.int32, torch.int64):
            src = sk.BitSource(77)
            x = torch.arange(70_001, dtype=dt, device="cuda")
            sk.merge(x, sk.MergeRange(1, 40_000, 30_000), src)
            a = np.arange(70_001, dtype=np.int64)
            st = O.state_vec(77, 0, 0, 0)
            O.merge(a, 1, 40_001, 70_001, st)
            assert np.array_equal(x.cpu().numpy().astype(np.int64), a)
    finally:
        lib.sk_debug_set(key, off)


@pytest.mark.parametrize("n,cutoff,seed,dt", [((1 << 25) + 17, 65536, 3, np.uint32), (1 << 24, 4096, 4, np.int64),
                                              (50_000_001, 65536, 5, np.float32),
                                              # leaves above 65536 elements: the unchunked host path
                                              (1 << 24, 1 << 21, 6, np.uint32), ((1 << 24) + 3, 1 << 20, 7, np.int64),
                                              (1 << 24, 1 << 19, 8, np.uint32)])
def test_host_entry_pipelined(n, cutoff, seed, dt):
    # numpy arrays go through the C-ABI host entry, which pipelines the H2D
    # copy with the leaf stage and the chunk-local rounds for n >= 2^24
    idx, bits = O.merge_shuffle_perm(n, cutoff, seed, threads=8)
    payload = (np.arange(n, dtype=np.int64) * 7 + 3).astype(dt)
    a = payload.copy()
    rep = sk.merge_shuffle_parallel(a, sk.ShuffleConfig(cutoff=cutoff), sk.BitSource(seed))
    assert rep.bits == bits
    assert np.array_equal(a, payload[idx])


@pytest.mark.parametrize("world,n,dt", [(2, (1 << 20) + 12345, torch.int32), (4, 1 << 21, torch.int64),
                                        (8, 3_000_001, torch.int32)])
def test_merge_shuffle_multi_single_process(world, n, dt):
    # the single-process multi-GPU entry (sk_merge_shuffle_multi), shards as
    # separate buffers (all on this device): host thread per shard, fused
    # peer-memory merge for the spanning rounds
    from paper_1508_03167_b200 import distributed as D
    cutoff, seed = 32768, 29
    shards = []
    for r in range(world):
        lo, hi = D.shard_range(n, cutoff, world, r)
        shards.append(torch.arange(lo, hi, dtype=dt, device="cuda"))
    bits = D.merge_shuffle_multi(shards, n, cutoff, seed)
    ref, rbits = O.merge_shuffle_perm(n, cutoff, seed)
    assert bits == rbits
    assert np.array_equal(torch.cat(shards).cpu().numpy().astype(np.int64), ref)


@pytest.mark.parametrize("variant", ["v3", "fallback", "quadratic"])
def test_leaf_apply_variants(variant):
    # leaves of 8193..65536 elements: the one-pass byte-counter kernel (v3)
    # and its serial fallback (counter overflow, forced for every leaf): same
    # permutations
    import ctypes
    from paper_1508_03167_b200 import _lib
    lib = _lib.load()
    lib.sk_debug_set.argtypes = [ctypes.c_int, ctypes.c_int]
    # quadratic: v3 with every bucket of >= 9 steps through the O(k^2) path
    knobs = {"v3": [], "fallback": [(6, 1)], "quadratic": [(1, 12)]}[variant]
    for k, v in knobs:
        lib.sk_debug_set(k, v)
    try:
        cases = [(1 << 20, 65536, 0), (1_000_000, 65536, 7), (300_007, 16384, 1234), (65536, 65536, 5),
                 (65535, 65536, 6), (40_000, 10_000, 8), (8193 * 2, 8193, 9)]
        if variant == "fallback":
            cases = cases[2:]
        for n, cutoff, seed in cases:
            for dt in (torch.int32, torch.int64):
                x, rep = gpu_perm(n, cutoff, seed, dt)
                ref, rbits = O.merge_shuffle_perm(n, cutoff, seed)
                assert rep.bits == rbits
                assert np.array_equal(x.cpu().numpy().astype(np.int64), ref), (n, cutoff, seed, dt)
    finally:
        lib.sk_debug_set(6, 0)
        lib.sk_debug_set(1, 99)


def test_more_than_65535_pairs_in_a_round():
    # n = 2^22 at cutoff 16: 2^18 leaves, 131072 pairs in round 1 (the tree
    # merge's transposed launch grid: pairs along x)
    for dt in (torch.int32, torch.int64):
        x, rep = gpu_perm(1 << 22, 16, 21, dt)
        ref, rbits = O.merge_shuffle_perm(1 << 22, 16, 21)
        assert rep.bits == rbits
        assert np.array_equal(x.cpu().numpy().astype(np.int64), ref)
