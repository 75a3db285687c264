#!/usr/bin/env python
"""Build A/B variants of one source file of libgscache.so (scratch measurement tooling).

  tools/ab_build.py <name> <source.cu> [file with the variant source]   -> ab/<name>/libgscache.so

The other objects come from the current build (paper_2502_14938_b200/build_obj); the variant is
compiled with the same flags.  tools/stage_profile.py loads a variant with GSC_AB_LIB=<path>.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_2502_14938_b200"))
import build as B  # noqa: E402


def main():
    name, src = sys.argv[1], sys.argv[2]
    text_file = sys.argv[3] if len(sys.argv) > 3 else os.path.join(B.CSRC, src)
    B.build()
    out = os.path.join(ROOT, "ab", name)
    os.makedirs(out, exist_ok=True)
    tmp_src = os.path.join(B.CSRC, "_ab_" + src)
    with open(text_file) as fh, open(tmp_src, "w") as gh:
        gh.write(fh.read())
    try:
        obj = os.path.join(out, src + ".o")
        subprocess.check_call([B.NVCC, *[f for f in B.NVCC_FLAGS if f not in ("-Xptxas", "-v")], "-c", tmp_src, "-o", obj])
    finally:
        os.unlink(tmp_src)
    objs = [obj if s == src else os.path.join(B.OBJ, s + ".o") for s in B.SOURCES]
    subprocess.check_call([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
                           "-o", os.path.join(out, "libgscache.so"), *objs])
    print(os.path.join(out, "libgscache.so"))


if __name__ == "__main__":
    main()
