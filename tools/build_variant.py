"""Build a variant of libmagicpig.so with extra nvcc defines into ablib/ (for A/B runs via MAGICPIG_LIB).
  python tools/build_variant.py NAME -DMP_EST_WARPS=10 ..."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_16179_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(b.ROOT, "ablib", name)
os.makedirs(out, exist_ok=True)


def one(src):
    obj = os.path.join(out, src.replace(".cu", ".o"))
    r = subprocess.run([b.NVCC, *b.FLAGS, *defs, "-c", os.path.join(b.CSRC, src), "-o", obj], capture_output=True,
                       text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    return obj


with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(one, b.SOURCES))
lib = os.path.join(out, "libmagicpig.so")
subprocess.run([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs, "-lcudart"],
               check=True)
print(lib)
