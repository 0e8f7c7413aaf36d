"""The C-ABI library builds/loads and exports every symbol include/*.h declares
(no compute calls: runs without a GPU)."""
import ctypes
import glob
import os
import re

from paper_1508_03167_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"\b(sk_[a-z0-9_]+)\s*\(", txt):
            names.add(m.group(1))
    return names


def test_library_exports_header_symbols():
    lib = _lib.load()
    names = declared_symbols()
    assert {"sk_merge_shuffle_parallel", "sk_fy_range", "sk_merge_range", "sk_chi_counts"} <= names
    for n in names:
        assert hasattr(lib, n), n
    assert set(_lib.SIGNATURES) == names


def test_version_and_error_string():
    lib = _lib.load()
    assert lib.sk_version() == 1
    assert isinstance(lib.sk_last_error(), bytes)


def test_invalid_arguments_rejected_without_gpu():
    lib = _lib.load()
    st = _lib.state_array((1, 0, 0, 0))
    assert lib.sk_merge_shuffle_parallel(None, 3, 10, 0, 0, None, None) == -1   # elem_bytes
    assert lib.sk_fy_range(None, 4, 5, 2, st, None) == -1                          # hi < lo
    assert lib.sk_merge_range(None, 4, 0, 5, 2, st, None) == -1                   # l < k
    assert lib.sk_chi_counts(7, 6, 10, 0, 0, None, None) == -1                     # algo
    assert lib.sk_balanced_shuffle(ctypes.c_void_p(16), 4, (1 << 20) + 1, st, None) == -1  # n above 2^20
