"""Build the native libraries in-tree (they travel to the GPU box with the snapshot).

  paper_2505_03269_b200/lib/libtcbf.so   the C-ABI library (include/tcbf.h), sm_100a
  paper_2505_03269_b200/lib/libtcbf_peaks.so  tensor/ALU peak micro-benchmarks (PAPER.md:113-122 analogue)
  synth/libsynth.so                       device twin of the seeded input generator
  oracle/liboracle.so                     the CPU oracle (test infrastructure; built, not used here)
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared",
              "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd, log):
    proc = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + proc.stdout + proc.stderr)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ... (log {log})")


def _compile_objects(srcs, objdir, extra, jobs):
    """nvcc -c every translation unit in parallel (one process per file), return the objects."""
    import concurrent.futures as cf
    os.makedirs(objdir, exist_ok=True)
    hdrs = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "tcbf.h")]

    def one(src):
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        if _stale(obj, [src] + hdrs):
            flags = [f for f in NVCC_FLAGS if f != "-shared"]
            cmd = [_nvcc(), *ARCH, *flags, *extra, "-I", os.path.join(ROOT, "include"), "-I", CSRC,
                   "-c", "-o", obj, src]
            _run(cmd, obj[:-2] + ".log")
        return obj

    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        return list(ex.map(one, srcs))


def build_tcbf(force=False, dev=False):
    """libtcbf.so (product).  dev=True builds libtcbf_dev.so with the TCBF_DEV ablation switches
    (DESIGN.md §4 studies); the binding never loads it unless a tool points library_path at it."""
    os.makedirs(LIBDIR, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    srcs = [s for s in srcs if not s.endswith("peaks.cu")]
    name = "libtcbf_dev.so" if dev else "libtcbf.so"
    out = os.path.join(LIBDIR, name)
    objdir = os.path.join(LIBDIR, "obj_dev" if dev else "obj")
    if force:
        for o in glob.glob(os.path.join(objdir, "*.o")):
            os.remove(o)
    objs = _compile_objects(srcs, objdir, ["-DTCBF_DEV"] if dev else [], jobs=max(1, os.cpu_count() or 1))
    if force or _stale(out, objs):
        cmd = [_nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-o", out, *objs,
               "-cudart=static"]
        _run(cmd, os.path.join(LIBDIR, "build_" + name[:-3] + ".log"))
    return out


def build_peaks(force=False):
    src = os.path.join(CSRC, "peaks.cu")
    if not os.path.exists(src):
        return None
    out = os.path.join(LIBDIR, "libtcbf_peaks.so")
    if force or _stale(out, [src, os.path.join(CSRC, "ptx.cuh")]):
        cmd = [_nvcc(), *ARCH, *NVCC_FLAGS, "-I", CSRC, "-o", out, src, "-cudart=static"]
        _run(cmd, os.path.join(LIBDIR, "build_peaks.log"))
    return out


def build_synth(force=False):
    src = os.path.join(ROOT, "synth", "gen_dev.cu")
    out = os.path.join(ROOT, "synth", "libsynth.so")
    if force or _stale(out, [src]):
        cmd = [_nvcc(), *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-o", out, src,
               "-cudart=static"]
        _run(cmd, os.path.join(LIBDIR, "build_synth.log"))
    return out


def build_oracle(force=False):
    sys.path.insert(0, ROOT)
    import oracle  # test infrastructure: compiled here, never called by the product path
    return oracle.build(force=force)


def build_all(force=False):
    os.makedirs(LIBDIR, exist_ok=True)
    return [build_tcbf(force), build_peaks(force), build_synth(force), build_oracle(force)]


if __name__ == "__main__":
    if "--dev" in sys.argv:
        print(build_tcbf(force="--force" in sys.argv, dev=True))
    else:
        for p in build_all(force="--force" in sys.argv):
            print(p)
