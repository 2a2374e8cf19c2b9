"""A/B helper (measurement aid, not product code): build a variant of the
extension in which some csrc files are replaced, linking the other objects
of the last in-tree build (build/objs).  Load it with WJ_LIB=ab/<name>.so.

    python profiles/ab_variant.py NAME csrc_name=path/to/variant.cu ...
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2202_13538_b200 import build as B  # noqa: E402


def main():
    name, repl = sys.argv[1], dict(a.split("=", 1) for a in sys.argv[2:])
    objdir = os.path.join(ROOT, "build", "objs")
    out = os.path.join(ROOT, "ab")
    os.makedirs(out, exist_ok=True)
    flags = [f for f in B.FLAGS if f not in ("-shared", "-cudart", "static")]
    flags += os.environ.get("ABV_FLAGS", "").split()  # e.g. ABV_FLAGS=-maxrregcount=152
    objs = []
    for src in B.SOURCES:
        if src in repl:
            obj = os.path.join(out, f"{name}_{os.path.splitext(src)[0]}.o")
            # the variant compiles with the csrc include path (it may live anywhere)
            subprocess.run([B.NVCC, *flags, "-c", "-I", os.path.join(ROOT, "include"), "-I", B.CSRC, "-o", obj,
                            os.path.abspath(repl[src])], check=True)
            objs.append(obj)
        else:
            objs.append(os.path.join(objdir, os.path.splitext(src)[0] + ".o"))
    lib = os.path.join(out, name + ".so")
    subprocess.run([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o", lib,
                    *objs], check=True)
    print(lib)


if __name__ == "__main__":
    main()
