import ctypes, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1508_03167_b200 import _lib
lib = _lib.load()
n = 1 << 30
warm = torch.zeros(1, device="cuda"); torch.cuda.synchronize()
host = torch.randint(0, 1 << 30, (n,), dtype=torch.int32).pin_memory()
hp = ctypes.c_void_p(host.data_ptr())
st = torch.cuda.current_stream()
sp = ctypes.c_void_p(st.cuda_stream)
for _ in range(3):
    t0 = time.perf_counter()
    _lib.check(lib.sk_merge_shuffle_parallel_host(hp, 4, n, 65536, 0, None, sp))
    print("wall ms", (time.perf_counter() - t0) * 1e3, file=sys.stderr)
