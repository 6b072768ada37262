"""Dev tool: build a compile-time variant of libtcbf.so for an A/B (AB_LIB=... tools/ab_gemm.py).

    python tools/build_variant.py NAME SOURCE.cu [-DKNOB=VALUE ...] [--dev]

Recompiles one translation unit of csrc/ with the given defines, links it with the product
objects of every other unit (paper_2505_03269_b200/lib/obj, built first) and writes
build/libtcbf_NAME.so.  The product library is untouched.
"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_03269_b200 import build as B  # noqa: E402


def main():
    name, src = sys.argv[1], sys.argv[2]
    dev = "--dev" in sys.argv   # link against the TCBF_DEV objects (TCBF_DEBUG ablations honoured)
    defines = [a for a in sys.argv[3:] if a != "--dev"] + (["-DTCBF_DEV"] if dev else [])
    B.build_tcbf(dev=dev)
    objdir = os.path.join(ROOT, "build", "obj_" + name)
    os.makedirs(objdir, exist_ok=True)
    srcpath = os.path.join(B.CSRC, src)
    obj = os.path.join(objdir, src[:-3] + ".o")
    flags = [f for f in B.NVCC_FLAGS if f != "-shared"]
    subprocess.run([B._nvcc(), *B.ARCH, *flags, *defines, "-I", os.path.join(ROOT, "include"), "-I", B.CSRC,
                    "-c", "-o", obj, srcpath], check=True, capture_output=True)
    others = [o for o in glob.glob(os.path.join(B.LIBDIR, "obj_dev" if dev else "obj", "*.o"))
              if os.path.basename(o) != src[:-3] + ".o"]
    out = os.path.join(ROOT, "build", f"libtcbf_{name}.so")
    subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-o", out, obj,
                    *others, "-cudart=static"], check=True)
    print(out)


if __name__ == "__main__":
    main()
