"""Build the current csrc/ into build/variants/NAME.so (experiments: load it with
SK_LIB_PATH=build/variants/NAME.so).  Extra arguments (e.g. -DSK_WS_TRIPS=64)
are passed to nvcc."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1508_03167_b200 import build as b  # noqa: E402

name = sys.argv[1]
extra = sys.argv[2:]
out = os.path.join(ROOT, "build", "variants")
os.makedirs(out, exist_ok=True)
objs, procs = [], []
for src in b.SOURCES:
    obj = os.path.join(out, name + "_" + src.replace(".cu", ".o"))
    procs.append(subprocess.Popen([b.NVCC, *b.FLAGS, *extra, "-c", os.path.join(b.CSRC, src), "-o", obj]))
    objs.append(obj)
assert all(p.wait() == 0 for p in procs)
subprocess.check_call([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                       os.path.join(out, name + ".so"), *objs])
for o in objs:
    os.remove(o)
print(os.path.join(out, name + ".so"))
