"""F3: the B200 backend's CLI against the reference CLI's own outputs
(tests/golden/cli.json, made by tests/golden/make_cli_golden.py): identical
permutations, bit counts, CSV rows (wall time excepted) and chi-square
verdicts.  Usage-error behaviour runs on CPU."""
import os
import subprocess
import sys

import pytest

from golden import CLI

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_cli(argv, stdin=None):
    env = dict(os.environ)
    env.pop("SHUFFLEKIT_SEED", None)
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    return subprocess.run([sys.executable, "-m", "paper_1508_03167_b200.cli", *argv], input=stdin or "",
                          capture_output=True, text=True, env=env, timeout=600)


def blank_wall(stdout, argv):
    if argv[0] != "bench":
        return stdout
    lines = stdout.splitlines()
    out = [lines[0]]
    for ln in lines[1:]:
        f = ln.split(",")
        f[5] = "*"
        out.append(",".join(f))
    return "\n".join(out) + "\n"


@pytest.mark.gpu
@pytest.mark.parametrize("case", CLI, ids=lambda c: "_".join(c["argv"][:3]) + f"_{abs(hash(str(c['argv']))) % 997}")
def test_cli_matches_reference(case):
    p = run_cli(case["argv"], case["stdin"])
    assert p.returncode == case["rc"], p.stderr
    assert blank_wall(p.stdout, case["argv"]) == case["stdout"]
    assert p.stderr == case["stderr"]


@pytest.mark.parametrize("argv", [["shuffle", "--algo", "balanced", "--n", str((1 << 20) + 1), "--seed", "1"],
                                  ["verify", "--mode", "exact", "--algo", "merge", "--n", "4"],
                                  ["shuffle", "--algo", "merge", "--n", "-1", "--seed", "1"],
                                  ["bench", "--algos", "merge", "--sizes", "x", "--seed", "1"]])
def test_cli_usage_errors(argv):
    p = run_cli(argv)
    assert p.returncode == 2
