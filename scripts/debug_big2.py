"""Element positions >= 2^32: leaf stage of a 2^32 + 2^22 uint64 array, and
single leaves / single merges placed above 2^32 against the same task at 0."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1508_03167_b200 import _lib  # noqa: E402

lib = _lib.load()
S = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
n = (1 << 32) + (1 << 22)
q = 1 << 17
x = torch.arange(n, dtype=torch.int64, device="cuda")
bits = ctypes.c_uint64(0)
print("shard rc", lib.sk_merge_shuffle_shard(ctypes.c_void_p(x.data_ptr()), 8, n, 65536, 5, 0, q, 0,
                                             ctypes.byref(bits), S()), flush=True)
torch.cuda.synchronize()


def leaf_of(p):
    i = (p * q) // n
    return torch.where(((i + 1) * n) // q <= p, i + 1, i)


CH = 1 << 27
bad_pos = []
for i in range(0, n, CH):
    v = x[i:i + CH]
    p = torch.arange(i, i + v.numel(), dtype=torch.int64, device="cuda")
    b = leaf_of(p) != leaf_of(v)
    if bool(b.any()):
        bp = p[b]
        bad_pos.append((int(bp.min()), int(bp.max()), int(b.sum())))
print("bad ranges", bad_pos[:10], len(bad_pos), flush=True)
hi_part = x[1 << 32:(1 << 32) + 64].tolist()
print("x[2^32 ..+64]", hi_part, flush=True)
lf = int(leaf_of(torch.tensor([1 << 32], device="cuda")))
lo_l, hi_l = (lf * n) // q, ((lf + 1) * n) // q
print("leaf at 2^32:", lf, lo_l, hi_l, "values", x[lo_l:lo_l + 8].tolist(), x[hi_l - 4:hi_l + 4].tolist(), flush=True)
del x
torch.cuda.empty_cache()

# single leaf above 2^32 vs at 0
for lo in ((1 << 32) + 8, (1 << 32) - 1000):
    m = 65536
    big = torch.zeros(lo + m + 16, dtype=torch.int64, device="cuda")
    big[lo:lo + m] = torch.arange(m, dtype=torch.int64, device="cuda")
    small = torch.arange(m, dtype=torch.int64, device="cuda")
    st1 = (ctypes.c_uint64 * 4)(77, 0, 0, 0)
    st2 = (ctypes.c_uint64 * 4)(77, 0, 0, 0)
    r1 = lib.sk_fy_range(ctypes.c_void_p(big.data_ptr()), 8, lo, lo + m, st1, S())
    r2 = lib.sk_fy_range(ctypes.c_void_p(small.data_ptr()), 8, 0, m, st2, S())
    torch.cuda.synchronize()
    print("fy lo", lo, r1, r2, "equal", torch.equal(big[lo:lo + m], small), list(st1) == list(st2), flush=True)
    # merge above 2^32 vs at 0
    big[lo:lo + m] = torch.arange(m, dtype=torch.int64, device="cuda")
    small = torch.arange(m, dtype=torch.int64, device="cuda")
    st1 = (ctypes.c_uint64 * 4)(78, 0, 0, 0)
    st2 = (ctypes.c_uint64 * 4)(78, 0, 0, 0)
    r1 = lib.sk_merge_range(ctypes.c_void_p(big.data_ptr()), 8, lo, lo + 30000, lo + m, st1, S())
    r2 = lib.sk_merge_range(ctypes.c_void_p(small.data_ptr()), 8, 0, 30000, m, st2, S())
    torch.cuda.synchronize()
    print("merge lo", lo, r1, r2, "equal", torch.equal(big[lo:lo + m], small), list(st1) == list(st2), flush=True)
    del big, small
    torch.cuda.empty_cache()
