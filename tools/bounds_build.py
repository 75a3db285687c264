#!/usr/bin/env python
"""Build the bounds-checked debug library ab/bounds/libgscache.so: every source compiled with
-DGSC_BOUNDS_CHECK (device-side checks of the data-dependent indices that trap with a message; see
gsc_internal.cuh GSC_CHECK) -- the stand-in for compute-sanitizer memcheck on pools that do not offer it.
Run the GPU suite against it with GSC_AB_LIB=ab/bounds/libgscache.so (tests/conftest.py)."""
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2502_14938_b200"))
import build as B  # noqa: E402


def main():
    out = os.path.join(ROOT, "ab", "bounds")
    os.makedirs(out, exist_ok=True)
    flags = [f for f in B.NVCC_FLAGS if f not in ("-Xptxas", "-v")] + ["-DGSC_BOUNDS_CHECK"]

    def one(src):
        o = os.path.join(out, src + ".o")
        subprocess.check_call([B.NVCC, *flags, "-c", os.path.join(B.CSRC, src), "-o", o])
        return o

    with cf.ThreadPoolExecutor(max_workers=len(B.SOURCES)) as ex:
        objs = list(ex.map(one, B.SOURCES))
    so = os.path.join(out, "libgscache.so")
    subprocess.check_call([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
                           "-o", so, *objs])
    print(so)


if __name__ == "__main__":
    main()
