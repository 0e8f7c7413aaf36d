"""Stage timing experiment helper (not part of the product or the bench).

    python scripts/prof_run.py LOG2N STEPS [key=value ...] [--check]

Runs merge_shuffle_parallel on 2^LOG2N uint32 elements (cutoff 65536, seed 0)
STEPS times after 2 warm-ups, with the library's per-stage CUDA-event timing
on, and prints one JSON line: ms per step and per stage.  key=value pairs are
passed to sk_debug_set (internal performance knobs) before the run, e.g.
5=0 (leaf apply variant).  --check compares the bit count with the
reference's for n = 2^26 / 2^30.
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from paper_1508_03167_b200 import _lib  # noqa: E402

BITS = {20: 20642558, 26: 1724975486, 30: 31908987766}


def main():
    log2n, steps = int(sys.argv[1]), int(sys.argv[2])
    knobs = [a for a in sys.argv[3:] if "=" in a]
    lib = _lib.load()
    for kv in knobs:
        k, v = kv.split("=")
        assert lib.sk_debug_set(int(k), int(v)) == 0, kv
    n = 1 << log2n
    eb = 8 if "--u64" in sys.argv else 4
    x = torch.arange(n, dtype=torch.int64 if eb == 8 else torch.int32, device="cuda")
    st = torch.cuda.current_stream()
    sp = ctypes.c_void_p(st.cuda_stream)
    bits = ctypes.c_uint64(0)
    for _ in range(2):
        _lib.check(lib.sk_merge_shuffle_parallel(ctypes.c_void_p(x.data_ptr()), eb, n, 65536, 0, ctypes.byref(bits), sp))
    torch.cuda.synchronize()
    ok = None
    if "--check" in sys.argv and log2n in BITS:
        ok = bits.value == BITS[log2n]
    lib.sk_profile_enable(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        _lib.check(lib.sk_merge_shuffle_parallel(ctypes.c_void_p(x.data_ptr()), eb, n, 65536, 0, None, sp))
    e1.record(st)
    torch.cuda.synchronize()
    sm = (ctypes.c_double * 5)()
    lib.sk_profile_read(sm, None, 5)
    lib.sk_profile_enable(0)
    names = ["leaf_decode", "leaf_apply", "merge_rounds", "identity+tail", "final_copy"]
    print(json.dumps({"log2n": log2n, "eb": eb, "knobs": knobs, "ms_per_step": round(e0.elapsed_time(e1) / steps, 3),
                      "stages": {k: round(sm[i] / steps, 3) for i, k in enumerate(names)}, "bits_ok": ok}))


if __name__ == "__main__":
    main()
