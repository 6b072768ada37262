#!/usr/bin/env python
"""Small invocations of every kernel of libtcbf.so, for compute-sanitizer (SURVEY.md §5 sanitizer
pass; the multi-stage mbarrier / TMEM pipelines of PAPER.md:167 are what it guards).

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_cases.py [group]

Each case runs pack + beamform (or the raw / interleaved entry points) at a tiny shape and at a
ragged one (odd M/N/K, partial tiles, masked-store epilogues) and checks the result against the
oracle, so a sanitizer run that reports nothing also produced correct output.  Groups: f16, b1,
misc, all (default).
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: the check, never the path)
import paper_2505_03269_b200 as tcbf  # noqa: E402
import synth  # noqa: E402


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _srcs(M, N, K, B, seed, dist="uniform"):
    w = synth.to_interleaved(synth.generate(dist, seed, 0, B, M, K))
    x = synth.to_interleaved(synth.generate(dist, seed, 1, B, K, N))
    return w, x


def _f16_ok(y, ref):
    yc = y[:, 0].astype(np.float64) + 1j * y[:, 1]
    rc = ref[:, 0] + 1j * ref[:, 1]
    return np.linalg.norm(yc - rc) <= 2e-3 * np.linalg.norm(rc)


def run_case(name, prec, M, N, K, B, path="packed", env=None):
    for k in [k for k in os.environ if k.startswith("TCBF_")]:   # the previous case's overrides
        os.environ.pop(k, None)
    os.environ.update(env or {})
    w, x = _srcs(M, N, K, B, 17 + M + N + K)
    plan = tcbf.Plan(M, N, K, B, prec)
    wp = plan.pack(tcbf.WEIGHTS, _dev(w))
    if path == "raw":
        y = plan.beamform_raw(wp, _dev(x))
        kern = plan.raw_variant
    elif path == "f16i":
        y = plan.beamform_f16i(wp, _dev(x).half())
        kern = "f16_interleaved"
    else:
        y = plan.beamform(wp, plan.pack(tcbf.DATA, _dev(x)))
        kern = plan.variant
    torch.cuda.synchronize()
    y = y.cpu().numpy()
    if prec == "b1":
        ok = np.array_equal(y, oracle.cgemm_b1(w, x, 0, M, N, K, B))
    else:
        ok = _f16_ok(y, oracle.cgemm_f16(w, x, 0, M, N, K, B))
    print(f"{'ok  ' if ok else 'FAIL'} {name:28s} {prec} M={M} N={N} K={K} B={B} path={path} kernel={kern}",
          flush=True)
    return ok


CASES = {
    "f16": [
        ("f16_default_tiny", "f16", 8, 64, 32, 2, "packed", None),
        ("f16_default_ragged", "f16", 200, 300, 100, 3, "packed", None),
        ("f16_masked_store", "f16", 129, 77, 65, 2, "packed", None),
        ("f16_n64", "f16", 130, 60, 200, 2, "packed", None),
        ("f16_bk32_s4_e8", "f16", 200, 300, 100, 2, "packed", {"TCBF_F16_VARIANT": "0"}),
        ("f16_pair_n128", "f16", 300, 260, 600, 1, "packed", None),
        ("f16_pair_n256", "f16", 300, 260, 2100, 1, "packed", None),
        ("f16_fused_raw", "f16", 200, 300, 100, 3, "raw", None),
        ("f16_fused_raw_tiny", "f16", 8, 64, 32, 2, "raw", None),
        ("f16_fused_raw_multicast", "f16", 200, 256, 100, 3, "raw", None),
        ("f16_tmem_multi_unit", "f16", 70, 256, 100, 80, "raw", None),
        ("f16_tmem_odd_n_fallback", "f16", 70, 77, 40, 2, "raw", None),
        ("f16_tmem_no_multicast", "f16", 130, 300, 200, 3, "raw", {"TCBF_F16_MC": "0"}),
        ("f16_smaj_raw", "f16", 200, 300, 100, 3, "raw", {"TCBF_F16_FUSED": "smaj"}),
        ("f16_stream_conv", "f16", 32, 260, 700, 1, "raw", {"TCBF_FORCE_STREAM_CONV": "1"}),
        ("f16_stream_conv_split", "f16", 40, 128, 3000, 1, "raw", {"TCBF_FORCE_STREAM_CONV": "1"}),
        ("f16_interleaved_tmem", "f16", 200, 300, 100, 2, "f16i", None),
        ("f16_interleaved_tmem_multi_unit", "f16", 64, 512, 64, 40, "f16i", None),
        ("f16_interleaved_resident", "f16", 200, 300, 100, 2, "f16i", {"TCBF_F16I": "res"}),
        ("f16_interleaved_resident_mc", "f16", 130, 256, 200, 3, "f16i", {"TCBF_F16I": "res"}),
        ("f16_interleaved_streaming", "f16", 200, 300, 100, 2, "f16i", {"TCBF_F16I_STREAM": "1"}),
        ("f16_interleaved_long_k", "f16", 100, 132, 333, 1, "f16i", None),
    ],
    "b1": [
        ("b1_f4_tiny", "b1", 8, 64, 32, 2, "packed", {"TCBF_NO_SWAP": "1"}),
        ("b1_f4_ragged", "b1", 130, 200, 1000, 2, "packed", None),
        ("b1_f4_masked", "b1", 100, 129, 31, 2, "packed", None),
        ("b1_f4_short_k_rows", "b1", 200, 300, 500, 3, "packed", None),
        ("b1_f4_long_k_tma", "b1", 130, 96, 5000, 1, "packed", None),
        ("b1_f4_swap32", "b1", 17, 260, 700, 2, "packed", None),
        ("b1_f4_swap64", "b1", 48, 77, 600, 2, "packed", None),
        ("b1_i8", "b1", 130, 200, 1000, 2, "packed", {"TCBF_B1_KERNEL": "i8"}),
        ("b1_i8_split", "b1", 40, 77, 3000, 2, "packed", {"TCBF_B1_KERNEL": "i8", "TCBF_B1_SPLITS": "3"}),
        ("b1_popc", "b1", 70, 45, 300, 3, "packed", {"TCBF_B1_KERNEL": "popc"}),
        ("b1_bmma", "b1", 70, 45, 300, 3, "packed", {"TCBF_B1_KERNEL": "bmma"}),
        ("b1_raw_pack", "b1", 70, 45, 300, 3, "raw", None),
    ],
}


def misc():
    """steering kernel + the host pipeline (tcbf_beamform_host)."""
    M, N, K, B = 33, 63, 33, 3
    plan = tcbf.Plan(M, N, K, B, "f16")
    pos = torch.arange(K, dtype=torch.float64, device="cuda") * 0.5
    th = torch.linspace(-1.0, 1.0, M, dtype=torch.float64, device="cuda")
    fr = torch.full((B,), 1.0, dtype=torch.float64, device="cuda")
    wsrc = plan.steering_weights(pos, th, fr, 1.0)
    wp = plan.pack(tcbf.WEIGHTS, wsrc)
    _, x = _srcs(M, N, K, B, 5)
    ref = plan.beamform_raw(wp, _dev(x))   # the call tcbf_beamform_host makes per chunk
    xh = torch.from_numpy(x).pin_memory()
    oh = torch.empty(tuple(ref.shape), dtype=ref.dtype).pin_memory()
    plan.beamform_host(wp, xh, oh)
    ok = torch.equal(oh, ref.cpu())
    print(f"{'ok  ' if ok else 'FAIL'} host_pipeline_and_steering  M={M} N={N} K={K} B={B}", flush=True)
    return ok


def main():
    group = sys.argv[1] if len(sys.argv) > 1 else "all"
    torch.cuda.set_device(0)
    ok = True
    for g in ("f16", "b1"):
        if group in (g, "all"):
            for c in CASES[g]:
                ok &= run_case(*c)
    if group in ("misc", "all"):
        ok &= misc()
    print("ALL OK" if ok else "SOME CASES FAILED", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
