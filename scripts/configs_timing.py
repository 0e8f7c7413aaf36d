"""Time every BASELINE config's GPU workload on one B200 (records for DESIGN.md).

    python scripts/configs_timing.py
Prints one JSON line per config: median of 5 timed calls after 2 warm-ups
(CUDA events around the call; device-resident data unless noted).
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1508_03167_b200 as sk  # noqa: E402
from paper_1508_03167_b200 import verify as V  # noqa: E402


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def line(name, ms, n, **kw):
    print(json.dumps({"config": name, "ms": round(ms, 3), "Gelem/s": round(n / ms / 1e6, 2) if n else None, **kw}),
          flush=True)


# SK_KNOBS="key=value,..." sets internal performance knobs (sk_debug_set) for A/B runs
for kv in filter(None, os.environ.get("SK_KNOBS", "").split(",")):
    from paper_1508_03167_b200 import _lib
    k, v = kv.split("=")
    assert _lib.load().sk_debug_set(int(k), int(v)) == 0, kv

g = torch.Generator(device="cuda").manual_seed(7)
# 1. identity 2^20, default cutoff (bit-exact vs the reference golden in the tests)
x = torch.arange(1 << 20, dtype=torch.int32, device="cuda")
line("1: 2^20 identity u32", timed(lambda: sk.merge_shuffle_parallel(x, sk.ShuffleConfig(), sk.BitSource(0))), 1 << 20)
# 2. 2^26 uniform u32 + chi-square 10^7 trials at n=6 (cutoff 65536 and 1)
x = torch.randint(-2 ** 31, 2 ** 31 - 1, (1 << 26,), dtype=torch.int32, device="cuda", generator=g)
line("2: 2^26 uniform u32", timed(lambda: sk.merge_shuffle_parallel(x, sk.ShuffleConfig(), sk.BitSource(0))), 1 << 26)
for cut in (65536, 1):
    t0 = time.perf_counter()
    c = V.chi_counts("merge_parallel", 6, 10 ** 7, 0, cut)
    line(f"2: chi_counts n=6 10^7 trials cutoff {cut}", (time.perf_counter() - t0) * 1e3, None,
         wall=True, statistic=round(float(((c - c.sum() / 720) ** 2 / (c.sum() / 720)).sum()), 2))
# 3. 2^30 uniform u32 (the bench workload)
x = torch.randint(-2 ** 31, 2 ** 31 - 1, (1 << 30,), dtype=torch.int32, device="cuda", generator=g)
line("3: 2^30 uniform u32, 1 GPU", timed(lambda: sk.merge_shuffle_parallel(x, sk.ShuffleConfig(), sk.BitSource(0)),
                                         reps=3), 1 << 30)
del x
# 4. one GPU's share of config 4: 2^30 uint64 keys (8 GB)
x = torch.arange(1 << 30, dtype=torch.int64, device="cuda")
line("4: 2^30 u64 identity (one GPU's 8 GB shard size)",
     timed(lambda: sk.merge_shuffle_parallel(x, sk.ShuffleConfig(), sk.BitSource(0)), reps=3), 1 << 30)
del x
# 5. batched 65536 x 4096 u32 and Rao-Sandelius at 2^24 / 2^30
x = torch.arange(65536 * 4096, dtype=torch.int32, device="cuda").reshape(65536, 4096) % 4096
line("5: batched 65536 x 4096 u32", timed(lambda: sk.batched_shuffle(x, sk.ShuffleConfig(), 0)), 65536 * 4096)
del x
for lg in (24, 30):
    x = torch.arange(1 << lg, dtype=torch.int32, device="cuda")
    line(f"F2: rs_shuffle_parallel 2^{lg} u32",
         timed(lambda: sk.rs_shuffle_parallel(x, sk.ShuffleConfig(), sk.BitSource(0)), reps=3), 1 << lg)
    del x
# F1 (config 5 names BalancedShuffle): the largest sizes served (wall time of
# the call, which includes its host-side plan and uploads)
for lg in (14, 16, 17):
    x = torch.arange(1 << lg, dtype=torch.int32, device="cuda")

    def bal():
        sk.balanced_shuffle(x, sk.ShuffleConfig(), sk.BitSource(1))
    bal()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        bal()
    torch.cuda.synchronize()
    line(f"F1: balanced_shuffle 2^{lg} u32", (time.perf_counter() - t0) * 1e3 / 3, 1 << lg, wall=True)
    del x
