"""Compare scripts/bs_host_check.cu (the GPU stages run on the host) with
oracle/balanced_oracle.py for given sizes (debugging aid)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import balanced_oracle as BO  # noqa: E402

for n in [int(a) for a in sys.argv[1:]]:
    st = (n * 7 + 3, 0, 0, 0)
    ref = list(range(n))
    bits, _ = BO.balanced_shuffle(ref, st)
    out = subprocess.run(["/tmp/bs_host_check", str(n), *map(str, st)], capture_output=True, text=True, timeout=600)
    lines = out.stdout.split("\n")
    got = [int(v) for v in lines[1].split()] if len(lines) > 1 else []
    bad = next((i for i in range(n) if i >= len(got) or got[i] != ref[i]), None)
    print(n, "bits", lines[0], bits, "first mismatch", bad, out.stderr[-200:], flush=True)
