"""Peak micro-benchmarks (the paper's cudapeak analogue, Table I).

Runs every kind in paper_2505_03269_b200/csrc/peaks.cu (register / shared-memory only, no HBM
traffic) on the current GPU and prints one JSON object: the measured rate per kind in TeraOps/s
(2 ops per multiply-accumulate; binary MACs for the 1-bit kinds) and, for the 1-bit kinds, the
rate expressed as useful complex-beamforming TeraOps/s (8 ops per complex MAC):
the XOR form needs 4 real b1 products per complex MAC (useful = raw), the paper's AND form 8
(useful = raw / 2), the tensor-core kinds are real-valued (useful = raw).

Usage (GPU box):  python tools/peaks.py [--out gpurun_out/peaks.json]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2505_03269_b200", "lib", "libtcbf_peaks.so")

KINDS = {
    0: ("b1_mma_sync_and_popc", "m16n8k256 .b1 .and.popc (legacy mma.sync)", 0.5),
    1: ("b1_mma_sync_xor_popc", "m16n8k256 .b1 .xor.popc (legacy mma.sync)", 1.0),
    2: ("cuda_core_xor_popc", "LOP3 + POPC + IADD on the CUDA cores", 1.0),
    3: ("tcgen05_f16", "tcgen05.mma kind::f16 128x256x16, fp32 acc", 1.0),
    4: ("tcgen05_i8", "tcgen05.mma kind::i8 128x256x32, int32 acc", 1.0),
    5: ("tcgen05_mxf4", "tcgen05.mma kind::mxf4 block32 128x256x64, fp32 acc", 1.0),
    6: ("tcgen05_f16_ts_n64", "tcgen05.mma kind::f16 128x64x16, A from TMEM", 1.0),
    7: ("tcgen05_f16_ss_n128", "tcgen05.mma kind::f16 128x128x16, A and B from smem", 1.0),
    8: ("tcgen05_mxf4_ts_n64", "tcgen05.mma kind::mxf4 block32 128x64x64, A from TMEM", 1.0),
    9: ("tcgen05_mxf4_ss_n64", "tcgen05.mma kind::mxf4 block32 128x64x64, A and B from smem", 1.0),
    10: ("tcgen05_mxf4_ts_n128", "tcgen05.mma kind::mxf4 block32 128x128x64, A from TMEM", 1.0),
    11: ("tcgen05_f16_ts_n128", "tcgen05.mma kind::f16 128x128x16, A from TMEM", 1.0),
    12: ("tcgen05_f16_ts_radio_step", "kind::f16 N=128 + N=64 (negate B) + N=64, A from TMEM (radio K step)", 1.0),
    13: ("tcgen05_f16_ts_n32", "tcgen05.mma kind::f16 128x32x16, A from TMEM", 1.0),
    14: ("tcgen05_f16_ts_radio_step_32beams", "kind::f16 N=64 + 2 x N=32, A from TMEM (32-beam K step)", 1.0),
}
# iterations per warp / issuing thread: each launch runs ~5-50 ms
ITERS = {0: 4000, 1: 4000, 2: 20000, 3: 40000, 4: 40000, 5: 40000, 6: 80000, 7: 80000, 8: 80000, 9: 80000,
         10: 80000, 11: 80000, 12: 40000, 13: 160000, 14: 80000}


def clocks():
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw", "--format=csv,noheader"],
                             capture_output=True, text=True, timeout=20).stdout.strip()
        return out
    except Exception as e:  # noqa: BLE001
        return f"unavailable: {e}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--repeat", type=int, default=3)
    ap.add_argument("--kinds", default=None, help="comma-separated kind numbers (default: all)")
    args = ap.parse_args()
    kinds = [int(k) for k in args.kinds.split(",")] if args.kinds else list(KINDS)
    if not os.path.exists(LIB):
        sys.exit(f"{LIB} missing: run python -c 'import __graft_entry__ as g; g.build()'")
    lib = ctypes.CDLL(LIB)
    lib.tcbf_peak_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(ctypes.c_double)]
    lib.tcbf_peak_run.restype = ctypes.c_int
    res = {}
    for kind in kinds:
        name, desc, useful = KINDS[kind]
        best = None
        for _ in range(args.repeat):
            s, o = ctypes.c_double(), ctypes.c_double()
            rc = lib.tcbf_peak_run(kind, ITERS[kind], ctypes.byref(s), ctypes.byref(o))
            if rc != 0:
                raise RuntimeError(f"tcbf_peak_run({kind}) -> {rc}")
            tops = o.value / s.value / 1e12
            if best is None or tops > best[0]:
                best = (tops, s.value)
        res[name] = dict(desc=desc, tera_ops_per_s=round(best[0], 1), ms=round(best[1] * 1e3, 3),
                         useful_complex_tera_ops_per_s=round(best[0] * useful, 1))
        print(f"{name:24s} {best[0]:9.1f} TeraOps/s  ({best[1] * 1e3:.2f} ms)", file=sys.stderr)
    out = dict(peaks=res, clocks_after=clocks(), note="best of %d launches, CUDA events" % args.repeat)
    line = json.dumps(out)
    print(line)
    if args.out:
        os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
