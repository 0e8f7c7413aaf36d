"""Experiment: the 2^30 shuffle eager (C ABI per call) vs replayed from a CUDA graph
captured once (same call).  Prints ms per shuffle for both, alternating."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1508_03167_b200 import _lib  # noqa: E402

lib = _lib.load()
n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
x = torch.randint(0, 1 << 31, (n,), dtype=torch.int32, device="cuda")


def call(s):
    _lib.check(lib.sk_merge_shuffle_parallel(ctypes.c_void_p(x.data_ptr()), 4, n, 65536, 0, None,
                                             ctypes.c_void_p(s.cuda_stream)))


cur = torch.cuda.current_stream()
for _ in range(3):
    call(cur)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(cur)
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
        call(s)
torch.cuda.synchronize()
for _ in range(2):
    g.replay()
torch.cuda.synchronize()


def timeit(fn, k=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(cur)
    for _ in range(k):
        fn()
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


for rep in range(3):
    print("eager", round(timeit(lambda: call(cur)), 3), "graph", round(timeit(g.replay), 3), flush=True)
