"""Leaves near element 2^32 of an n = 2^32 + 2^22 array: a 64-leaf shard
(small buffer, big geometry) with the lane- and the warp-per-leaf decode,
against the oracle's leaves."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1508_03167_b200 import _lib  # noqa: E402
from oracle import oracle as O  # noqa: E402

lib = _lib.load()
lib.sk_debug_set.argtypes = [ctypes.c_int, ctypes.c_int]
S = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
n = (1 << 32) + (1 << 22)
c, q = 17, 1 << 17
seed = 5
bound = lambda i: (n * i) >> c  # noqa: E731
for blk0, nblk in ((130880, 64), (0, 64), (65536, 64), (131008, 64)):
    lo, hi = bound(blk0), bound(blk0 + nblk)
    ref = np.arange(lo, hi, dtype=np.int64)
    for i in range(blk0, blk0 + nblk):
        st = O.state_vec(O.substream_seed(seed, i), 0, 0, 0)
        O.fy_range(ref, bound(i) - lo, bound(i + 1) - lo, st)
    for knob in (0, 1 << 30):
        lib.sk_debug_set(7, knob)
        x = torch.arange(lo, hi, dtype=torch.int64, device="cuda")
        bits = ctypes.c_uint64(0)
        rc = lib.sk_merge_shuffle_shard(ctypes.c_void_p(x.data_ptr()), 8, n, 65536, seed, blk0, nblk, 0,
                                        ctypes.byref(bits), S())
        torch.cuda.synchronize()
        got = x.cpu().numpy()
        bad = np.nonzero(got != ref)[0]
        print(f"blk0={blk0} decode={'lane' if knob == 0 else 'warp'} rc={rc} bad={bad.size} "
              f"first={bad[:3].tolist()} got={got[bad[:3]].tolist()} ref={ref[bad[:3]].tolist()}", flush=True)
    lib.sk_debug_set(7, 4096)
