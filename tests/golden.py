"""Loader for the committed golden fixtures (generated from the unmodified
reference by tests/golden/make_golden.py)."""
import hashlib
import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
G = json.load(open(os.path.join(HERE, "golden.json")))
CHI = dict(np.load(os.path.join(HERE, "chi_n6.npz")))
CHI_STATS = json.load(open(os.path.join(HERE, "chi_stats.json")))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cutoff_of(case):
    return 65536 if case["cutoff"] is None else case["cutoff"]

CLI = json.load(open(os.path.join(HERE, "cli.json")))
RS = json.load(open(os.path.join(HERE, "rs.json")))
