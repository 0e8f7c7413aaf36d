"""Golden outputs of the UNMODIFIED reference CLI (`shufflekit` = cli.py).

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_cli_golden.py

Writes tests/golden/cli.json: for each command line, the reference's exit
code, stdout and stderr (wall-clock columns of `bench` are blanked).  The
commands only use algorithms the B200 backend serves (fy, merge, rs,
balanced for n <= 2^17; chisq for fy / merge / merge_parallel / balanced).
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

OUT = os.path.dirname(os.path.abspath(__file__))

TOKENS = "\n".join(f"tok{i:03d}" for i in range(57)) + "\n"

CASES = [
    {"argv": ["shuffle", "--algo", "merge", "--n", "20", "--seed", "7", "--threads", "2", "--report"]},
    {"argv": ["shuffle", "--algo", "merge", "--n", "1000", "--seed", "8", "--threads", "4", "--cutoff", "100"]},
    {"argv": ["shuffle", "--algo", "merge", "--n", "300", "--seed", "9", "--cutoff", "16", "--report"]},
    {"argv": ["shuffle", "--algo", "fy", "--n", "15", "--seed", "3", "--report"]},
    {"argv": ["shuffle", "--algo", "merge", "--seed", "11", "--threads", "3", "--report"], "stdin": TOKENS},
    {"argv": ["shuffle", "--algo", "fy", "--seed", "12"], "stdin": TOKENS},
    {"argv": ["bench", "--algos", "merge,fy", "--sizes", "100,1000,70000", "--trials", "5", "--seed", "1",
              "--threads", "2"]},
    {"argv": ["bench", "--algos", "merge", "--sizes", "0,1,2,5000", "--trials", "3", "--seed", "2",
              "--threads", "8", "--cutoff", "64"]},
    {"argv": ["shuffle", "--algo", "rs", "--n", "40000", "--seed", "21", "--threads", "4", "--report"]},
    {"argv": ["shuffle", "--algo", "rs", "--n", "500", "--seed", "22", "--cutoff", "8", "--report"]},
    {"argv": ["bench", "--algos", "rs,merge", "--sizes", "1000,50000", "--trials", "3", "--seed", "5",
              "--threads", "2"]},
    {"argv": ["verify", "--mode", "chisq", "--algo", "merge_parallel", "--n", "5", "--trials", "20000", "--seed",
              "2", "--cutoff", "1"]},
    {"argv": ["verify", "--mode", "chisq", "--algo", "fy", "--n", "4", "--trials", "5000", "--seed", "3"]},
    # BalancedShuffle, the n <= 32 slice the B200 backend serves
    {"argv": ["shuffle", "--algo", "balanced", "--n", "20", "--seed", "3", "--report"]},
    {"argv": ["shuffle", "--algo", "balanced", "--seed", "13", "--report"], "stdin": "\n".join(f"w{i}" for i in range(29)) + "\n"},
    {"argv": ["bench", "--algos", "balanced,merge", "--sizes", "5,17,32", "--trials", "4", "--seed", "2",
              "--threads", "2"]},
    {"argv": ["verify", "--mode", "chisq", "--algo", "balanced", "--n", "4", "--trials", "5000", "--seed", "3"]},
    # BalancedShuffle with multi-limb ranks (n > 32)
    {"argv": ["shuffle", "--algo", "balanced", "--n", "100", "--seed", "4", "--report"]},
    {"argv": ["bench", "--algos", "balanced", "--sizes", "33,1000,5000", "--trials", "2", "--seed", "6",
              "--threads", "1"]},
]


def blank_wall(stdout: str, argv) -> str:
    if argv[0] != "bench":
        return stdout
    lines = stdout.splitlines()
    out = [lines[0]]
    for ln in lines[1:]:
        f = ln.split(",")
        f[5] = "*"  # mean_wall_ns
        out.append(",".join(f))
    return "\n".join(out) + "\n"


def main():
    res = []
    env = dict(os.environ)
    env.pop("SHUFFLEKIT_SEED", None)
    for c in CASES:
        p = subprocess.run([sys.executable, "-m", "shufflekit.cli", *c["argv"]], input=c.get("stdin", ""),
                           capture_output=True, text=True, env=env, timeout=600)
        res.append({"argv": c["argv"], "stdin": c.get("stdin"), "rc": p.returncode,
                    "stdout": blank_wall(p.stdout, c["argv"]), "stderr": p.stderr})
        print(c["argv"], p.returncode, len(p.stdout), file=sys.stderr)
    with open(os.path.join(OUT, "cli.json"), "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
