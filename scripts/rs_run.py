"""Rao-Sandelius at 2^LOG2N uint32 (timing / profiling helper): python scripts/rs_run.py LOG2N REPS"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1508_03167_b200 as sk  # noqa: E402

lg, reps = int(sys.argv[1]), int(sys.argv[2])
x = torch.arange(1 << lg, dtype=torch.int32, device="cuda")
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sk.rs_shuffle_parallel(x, sk.ShuffleConfig(), sk.BitSource(0))
    torch.cuda.synchronize()
    print("rs ms", round((time.perf_counter() - t0) * 1e3, 2), file=sys.stderr)
