"""Localise a failure above 2^32 elements: shuffle n = 2^32 + 2^22 uint64
identity keys with the leaves and rounds 1..k only (sk_merge_shuffle_shard
on the whole array) and check after each k that the result is a permutation
and that every element stayed inside its round-k pair."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1508_03167_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 32) + (1 << 22)
ks = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else list(range(0, 18))
cutoff, seed = 65536, 5
c = 0
while (n >> c) > cutoff:
    c += 1
q = 1 << c
lib = _lib.load()
CH = 1 << 27


def leaf_of(p):
    i = (p * q) // n
    return torch.where(((i + 1) * n) // q <= p, i + 1, i)


for k in ks:
    x = torch.arange(n, dtype=torch.int64, device="cuda")
    bits = ctypes.c_uint64(0)
    t0 = time.time()
    rc = lib.sk_merge_shuffle_shard(ctypes.c_void_p(x.data_ptr()), 8, n, cutoff, seed, 0, q, k, ctypes.byref(bits),
                                    ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    if rc:
        print("k", k, "rc", rc, lib.sk_last_error())
        break
    seen = torch.zeros(n, dtype=torch.bool, device="cuda")
    bad_group = 0
    lo_v, hi_v = 1 << 62, -1
    for i in range(0, n, CH):
        v = x[i:i + CH]
        lo_v, hi_v = min(lo_v, int(v.min())), max(hi_v, int(v.max()))
        if lo_v < 0 or hi_v >= n:
            break
        seen[v] = True
        p = torch.arange(i, i + v.numel(), dtype=torch.int64, device="cuda")
        bad_group += int((leaf_of(p) >> k != leaf_of(v) >> k).sum())
    perm = lo_v >= 0 and hi_v < n and bool(seen.all())
    miss = int((~seen).sum()) if lo_v >= 0 and hi_v < n else -1
    print(f"k={k} bits={bits.value} perm={perm} missing={miss} out_of_group={bad_group} "
          f"range=[{lo_v},{hi_v}] head={x[:4].tolist()} t={time.time() - t0:.1f}s", flush=True)
    del x, seen
    torch.cuda.empty_cache()
