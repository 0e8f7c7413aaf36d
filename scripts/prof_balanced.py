"""One BalancedShuffle of n elements (for an ncu launch list)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1508_03167_b200 as sk  # noqa: E402

n = int(sys.argv[1])
x = torch.arange(n, dtype=torch.int32, device="cuda")
sk.balanced_shuffle(x, sk.ShuffleConfig(), sk.BitSource(1))
torch.cuda.synchronize()
