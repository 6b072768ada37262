"""SASS instruction census of the kernels in libtcbf.so (cuobjdump -sass), proving which hardware
paths each kernel uses: tcgen05 MMAs (UTCHMMA = kind::f16, UTCIMMA = kind::i8, UTCOMMA = kind::mxf4 block-scaled fp4),
TMEM loads/stores (LDTM / STTM), TMA (UTMALDG loads, UTMASTG stores, UTMAREDG reduce-add), plain
global stores (STG), warp shuffles (SHFL), legacy mma.sync (HMMA / IMMA) and popcounts (POPC).

    python tools/sass_census.py [lib] > profiles/r02/sass_census.md
"""
import os
import re
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTCHMMA", "UTCIMMA", "UTCOMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMAREDG", "UBLKCP", "STG", "LDG",
        "STS", "LDS", "SHFL", "HMMA", "IMMA", "POPC", "SYNCS", "F2FP", "REDG", "CALL"]


def demangle(names):
    p = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return p.stdout.splitlines() if p.returncode == 0 else names


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2505_03269_b200", "lib", "libtcbf.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and cur:
            funcs[cur][m.group(1)] += 1
    names = list(funcs)
    pretty = demangle(names)
    print(f"# SASS census of `{os.path.relpath(lib, ROOT)}` (cuobjdump -sass, sm_100a)\n")
    print("Static instruction counts per kernel (not executed counts).\n")
    print("| kernel | " + " | ".join(KEYS) + " |")
    print("|---" * (len(KEYS) + 1) + "|")
    for n, p in zip(names, pretty):
        p = re.sub(r"tcbf::\(anonymous namespace\)::", "", p)
        p = re.sub(r"\(CUtensorMap_st.*|\(tcbf::Gemm.*", "", p)
        print(f"| `{p}` | " + " | ".join(str(funcs[n][k]) if funcs[n][k] else "" for k in KEYS) + " |")


if __name__ == "__main__":
    main()
