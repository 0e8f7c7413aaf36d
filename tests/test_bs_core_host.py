"""The serial multi-limb BalancedShuffle stages (csrc/bs_core.cuh: exact class
sizes, the fast dice roll on limbs, the recursive-halving unranking) built as
a HOST program (scripts/bs_host_check.cu, a debugging harness -- the product
runs the same source on the GPU) and compared with the Python-integer oracle,
which is pinned to the reference's goldens (test_oracle_balanced_big.py).
Runs without a GPU (nvcc compiles the host code)."""
import os
import shutil
import subprocess

import pytest

from oracle import balanced_oracle as BO

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


@pytest.fixture(scope="module")
def harness(tmp_path_factory):
    if not (os.path.exists(NVCC) or shutil.which("nvcc")):
        pytest.skip("nvcc not available")
    exe = str(tmp_path_factory.mktemp("bs") / "bs_host_check")
    subprocess.check_call([NVCC, "-O2", "-std=c++17", "-I", os.path.join(ROOT, "paper_1508_03167_b200", "csrc"),
                           os.path.join(ROOT, "scripts", "bs_host_check.cu"), "-o", exe],
                          stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    return exe


@pytest.mark.parametrize("n,state", [(33, (5, 0, 0, 0)), (64, (7, 0, 0, 0)), (100, (11, 0, 0, 0)),
                                     (257, (13, 0, 0, 0)), (1000, (17, 0, 0, 0)), (2049, (19, 0, 0, 0)),
                                     (5000, (23, 0, 0, 0)), (300, "mid")])
def test_host_stages_match_oracle(harness, n, state):
    if state == "mid":  # a mid-stream source: 37 bits taken, 27 of a word buffered
        s = BO.Stream((29, 0, 0, 0))
        s.bits(37)
        state = s.state()
    out = subprocess.run([harness, str(n), *map(str, state)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.split("\n")
    ref = list(range(n))
    bits, _ = BO.balanced_shuffle(ref, state)
    assert int(lines[0]) == bits
    assert [int(v) for v in lines[1].split()] == ref
