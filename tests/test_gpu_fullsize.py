"""Whole-array parity at the headline sizes (BASELINE configs 3 and 4).

* n = 2^30, 2^31 and 3*2^29+7: the SHA-256 of the ENTIRE permuted identity,
  as uint32 and uint64, equals the unmodified reference's
  (tests/golden/big.json, made by tests/golden/make_big_golden.py from
  merge_shuffle_parallel, shufflers.py:251-299), with its bit count.
* n = 2^33 uint64 (config 4, 64 GB) on ONE B200: the single-GPU path and the
  8-shard schedule with every shard on this device (sk_merge_shuffle_multi:
  a host thread per shard, spanning rounds as the fused peer-memory merge)
  produce the same array (device fingerprint) and bit count, and the result
  is a permutation of 0..n-1 (every key seen exactly once).  Bit-exactness of
  that code path against the reference is pinned at 2^24 by
  test_gpu_parity.test_config4_sharded_2p24_uint64_golden.
"""
import hashlib
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1508_03167_b200 as sk  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
BIG = json.load(open(os.path.join(HERE, "big.json")))["cases"]
CHUNK = 1 << 27


def device_sha(x: torch.Tensor) -> str:
    """SHA-256 of the tensor's little-endian bytes, streamed through host chunks."""
    h = hashlib.sha256()
    flat = x.view(-1)
    for i in range(0, flat.numel(), CHUNK):
        h.update(flat[i:i + CHUNK].cpu().numpy().tobytes())
    return h.hexdigest()


def fingerprint(x: torch.Tensor, offset: int = 0) -> int:
    """Position-weighted, nonlinear 64-bit fingerprint computed on the device
    (wrapping int64 arithmetic; additive over parts at their global offsets):
    any difference in any element changes it w.h.p."""
    acc = torch.zeros((), dtype=torch.int64, device=x.device)
    for i in range(0, x.numel(), CHUNK):
        v = x[i:i + CHUNK].to(torch.int64)
        pos = torch.arange(offset + i, offset + i + v.numel(), dtype=torch.int64, device=x.device)
        v = v * -7046029254386353131 + pos          # G as a signed int64
        v = v ^ (v >> 31)
        v = v * -4658895280553007687                # MIX1 as a signed int64
        acc += (v ^ (v >> 29)).sum()
    return int(acc.item())


def release_device_memory() -> None:
    """Return torch's cached blocks and the library's stream-ordered pool
    (it keeps freed memory for the next call) to the driver."""
    from cuda.bindings import runtime as rt
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    err, pool = rt.cudaDeviceGetDefaultMemPool(torch.cuda.current_device())
    assert err == rt.cudaError_t.cudaSuccess
    rt.cudaMemPoolTrimTo(pool, 0)


def identity(n: int, dtype) -> torch.Tensor:
    """0..n-1 on the device, built in chunks: torch 2.11's CUDA arange writes
    zeros past element 2^32 (measured on the B200 box: scripts/debug_arange.py)."""
    x = torch.empty(n, dtype=dtype, device="cuda")
    for i in range(0, n, CHUNK):
        x[i:i + CHUNK] = torch.arange(i, min(n, i + CHUNK), dtype=dtype, device="cuda")
    return x


def _mixed(v: torch.Tensor) -> torch.Tensor:
    v = v.to(torch.int64) * -7046029254386353131 + 0x2545F491
    v = v ^ (v >> 29)
    v = v * -4658895280553007687
    return v ^ (v >> 32)


def is_permutation(x: torch.Tensor) -> bool:
    """Every value in [0, n) exactly once: all values in range, and the
    order-independent multiset hash sum(mixed(v)) equals that of 0..n-1 (a
    repeated or missing value changes it w.h.p.)."""
    n = x.numel()
    got = torch.zeros((), dtype=torch.int64, device=x.device)
    want = torch.zeros((), dtype=torch.int64, device=x.device)
    for i in range(0, n, CHUNK):
        c = x[i:i + CHUNK].to(torch.int64)
        if int(c.min()) < 0 or int(c.max()) >= n:
            return False
        got += _mixed(c).sum()
        want += _mixed(torch.arange(i, i + c.numel(), dtype=torch.int64, device=x.device)).sum()
    return int(got) == int(want)


@pytest.mark.parametrize("case", BIG, ids=lambda c: f"n{c['n']}_s{c['seed']}")
@pytest.mark.parametrize("dtype", [torch.int32, torch.int64])
def test_whole_array_sha_against_reference(case, dtype):
    n = case["n"]
    x = identity(n, dtype)
    rep = sk.merge_shuffle_parallel(x, sk.ShuffleConfig(), sk.BitSource(case["seed"]))
    assert rep.bits == case["bits"]
    assert x[:8].cpu().tolist() == case["head"] and x[-2:].cpu().tolist() == case["tail"]
    assert device_sha(x) == case["sha_u32" if dtype == torch.int32 else "sha_u64"]
    del x
    release_device_memory()


def test_config4_2p33_uint64_one_gpu_equals_8_shards():
    n, seed = 1 << 33, 0
    release_device_memory()
    free, _ = torch.cuda.mem_get_info()
    if free < 170 * (1 << 30):
        pytest.skip(f"needs ~170 GB of free device memory, have {free / 2**30:.0f} GiB")
    x = identity(n, torch.int64)
    assert is_permutation(x) and int(x[-1]) == n - 1
    rep = sk.merge_shuffle_parallel(x, sk.ShuffleConfig(), sk.BitSource(seed))
    fp1, bits1 = fingerprint(x), rep.bits
    assert is_permutation(x)
    assert not torch.equal(x[:1 << 20], torch.arange(1 << 20, dtype=torch.int64, device="cuda"))
    del x
    release_device_memory()
    from paper_1508_03167_b200 import distributed as D
    shards = []
    for r in range(8):
        lo, hi = D.shard_range(n, 65536, 8, r)
        shards.append(torch.arange(lo, hi, dtype=torch.int64, device="cuda"))
    bits8 = D.merge_shuffle_multi(shards, n, 65536, seed)
    assert bits8 == bits1
    fp8, off = 0, 0
    for t in shards:
        fp8 += fingerprint(t, off)
        off += t.numel()
    assert (fp8 - fp1) % (1 << 64) == 0
    del shards
    release_device_memory()
