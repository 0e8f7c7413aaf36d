"""Stage timing of the batched config (BASELINE config 5): B arrays of L uint32.

    python scripts/prof_batched.py [B] [L] [steps] [key=value ...]
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1508_03167_b200 import _lib  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
L = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
lib = _lib.load()
for kv in [a for a in sys.argv[4:] if "=" in a]:
    k, v = kv.split("=")
    assert lib.sk_debug_set(int(k), int(v)) == 0
x = torch.arange(B * L, dtype=torch.int32, device="cuda") % L
st = torch.cuda.current_stream()
sp = ctypes.c_void_p(st.cuda_stream)
for _ in range(2):
    _lib.check(lib.sk_batched_shuffle(ctypes.c_void_p(x.data_ptr()), 4, B, L, 65536, 0, None, sp))
torch.cuda.synchronize()
lib.sk_profile_enable(1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(steps):
    _lib.check(lib.sk_batched_shuffle(ctypes.c_void_p(x.data_ptr()), 4, B, L, 65536, 0, None, sp))
e1.record(st)
torch.cuda.synchronize()
sm = (ctypes.c_double * 5)()
lib.sk_profile_read(sm, None, 5)
ms = e0.elapsed_time(e1) / steps
print(json.dumps({"B": B, "L": L, "ms": round(ms, 3), "Gelem/s": round(B * L / ms / 1e6, 2),
                  "decode": round(sm[0] / steps, 3), "apply": round(sm[1] / steps, 3)}))
