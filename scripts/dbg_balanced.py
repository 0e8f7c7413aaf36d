"""Debug helper: GPU BalancedShuffle vs the oracle for given sizes (prints
the first mismatch)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1508_03167_b200 as sk  # noqa: E402
from oracle import balanced_oracle as BO  # noqa: E402

for n in [int(a) for a in sys.argv[1:]]:
    src = sk.BitSource(n)
    ref = list(range(n))
    bits, st = BO.balanced_shuffle(ref, src.state_tuple())
    x = torch.arange(n, dtype=torch.int64, device="cuda")
    t0 = time.perf_counter()
    rep = sk.balanced_shuffle(x, sk.ShuffleConfig(), src)
    dt = time.perf_counter() - t0
    got = x.cpu().tolist()
    bad = next((i for i in range(n) if got[i] != ref[i]), None)
    print(n, "ms", round(dt * 1e3, 1), "bits", rep.bits, bits, "first mismatch", bad, flush=True)
